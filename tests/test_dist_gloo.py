"""Multi-process (world size 2, gloo, CPU) coverage of the N>1 protocol of tcl_topk_global:
contiguous candidate shards with global indices (libtcl's tcl_shard_range), the packed
(score, index) keys every rank computes (libtcl's tcl_topk_key, the encoding the device kernels
use), all-gather of each rank's best k keys, and the merge -> the identical global top-k on every
rank, equal to the top-k of the whole batch.  The device halves of the same protocol
(tcl_topk_local_keys / tcl_topk_merge_keys) are covered on the GPU by tests/test_gpu_multi.py."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import inputs


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _merge_keys(keys, k):
    """Best k of packed uint64 keys (descending), decoded: idx = 0xFFFFFFFF - low word."""
    u = np.sort(np.asarray(keys, dtype=np.int64).view(np.uint64))[::-1][:k]
    u = u[u != 0]                                  # 0 = padding
    idx = (np.uint64(0xFFFFFFFF) - (u & np.uint64(0xFFFFFFFF))).astype(np.int64)
    return idx.tolist()


def _worker(rank, world, port, n, k, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import oracle as O
    from paper_2604_12891_b200.tcl import shard_range, topk_key
    c = inputs.config("tiny")
    d = c["dims"]
    w = inputs.make_weights(d, c["seed"])
    f, l = inputs.make_features(d, n, c["seed"] + 1)
    lo, cnt = shard_range(n, world, rank)          # libtcl host code
    s = O.score(d, w, f[lo:lo + cnt], l[lo:lo + cnt], nthreads=2).astype(np.float32)
    keys = np.array([topk_key(float(v), lo + i) for i, v in enumerate(s)], dtype=np.uint64)
    local = np.zeros(k, np.uint64)                 # this rank's best k keys, 0-padded
    best = np.sort(keys)[::-1][:k]
    local[:best.size] = best
    gk = [torch.zeros(k, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(gk, torch.from_numpy(local.view(np.int64)))
    merged = _merge_keys(torch.cat(gk).numpy(), k)
    out_q.put((rank, merged, s.tolist(), lo))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("n,k", [(300, 16), (37, 64)])
def test_global_topk_protocol_world2(oracle, n, k):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n, k, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    assert res[0][1] == res[1][1]                  # identical on every rank
    s_all = np.zeros(n, np.float32)
    for _, _, s, lo in res:
        s_all[lo:lo + len(s)] = s
    gi, _ = oracle.topk(s_all, k)
    assert res[0][1] == [i for i in gi.tolist() if i >= 0]


def test_topk_key_order_matches_lexsort():
    """Sorting libtcl's packed keys descending == (score desc, index asc), NaN = -inf, -0 == +0."""
    from paper_2604_12891_b200.tcl import topk_key
    rng = np.random.default_rng(0)
    s = np.round(rng.standard_normal(500), 1).astype(np.float32)
    s[[3, 9]] = np.nan
    s[[4, 5]] = [-0.0, 0.0]
    s[[6, 7]] = [np.inf, -np.inf]
    keys = np.array([topk_key(float(v), 1000 + i) for i, v in enumerate(s)], dtype=np.uint64)
    order = np.argsort(keys)[::-1]
    key = np.where(np.isnan(s), -np.inf, s).astype(np.float64)
    key[key == 0] = 0.0
    assert np.array_equal(order, np.lexsort((np.arange(500), -key)))
    assert topk_key(1.0, 0) != 0 and topk_key(float("-inf"), 0xFFFFFFFF - 1) != 0


def test_shard_range_partitions():
    from paper_2604_12891_b200.tcl import shard_range
    for n in (0, 1, 7, 65536, 1048577):
        for world in (1, 2, 3, 8):
            parts = [shard_range(n, world, r) for r in range(world)]
            covered = []
            for st, cnt in parts:
                covered += list(range(st, st + cnt)) if n < 100 else [st, st + cnt]
            if n < 100:
                assert covered == list(range(n))
            assert sum(c for _, c in parts) == n
