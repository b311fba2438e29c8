"""Multi-process (world size 2, gloo, CPU) coverage of the N>1 protocol of tcl_topk_global:
contiguous candidate shards with global indices, local top-k per rank, all-gather of the k
(index, score) pairs, and the merge -> the identical global top-k on every rank, equal to the
top-k of the whole batch.  The GPU kernels of the same protocol are covered by
tests/test_gpu_parity.py (NCCL with one rank, virtual shards)."""
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


def _worker(rank, world, port, n, k, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import oracle as O
    from paper_2604_12891_b200.tcl import shard_range
    c = inputs.config("tiny")
    d = c["dims"]
    w = inputs.make_weights(d, c["seed"])
    f, l = inputs.make_features(d, n, c["seed"] + 1)
    lo, cnt = shard_range(n, world, rank)
    s = O.score(d, w, f[lo:lo + cnt], l[lo:lo + cnt], nthreads=2).astype(np.float32)
    idx, top = O.topk(s, k, index_base=lo)
    gi = [torch.zeros(k, dtype=torch.int64) for _ in range(world)]
    gt = [torch.zeros(k, dtype=torch.float32) for _ in range(world)]
    dist.all_gather(gi, torch.from_numpy(idx))
    dist.all_gather(gt, torch.from_numpy(top))
    cat_i = torch.cat(gi).numpy()
    cat_t = torch.cat(gt).numpy()
    order = np.lexsort((np.where(cat_i < 0, np.iinfo(np.int64).max, cat_i), -cat_t.astype(np.float64)))[:k]
    out_q.put((rank, cat_i[order].tolist(), cat_t[order].tolist(), s.tolist(), lo))
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
    assert res[0][1] == res[1][1] and res[0][2] == res[1][2]       # identical on every rank
    s_all = np.zeros(n, np.float32)
    for _, _, _, s, lo in res:
        s_all[lo:lo + len(s)] = s
    gi, gt = oracle.topk(s_all, k)
    assert list(gi) == res[0][1]
    assert np.array_equal(np.array(res[0][2], np.float32), gt)


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
