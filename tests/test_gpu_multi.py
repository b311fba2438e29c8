"""Multi-GPU protocol on the GPU ("selects the best K").

tcl_topk_global = tcl_topk_local_keys (this rank's best k as packed keys) -> ncclAllGather ->
tcl_topk_merge_keys.  This environment has ONE GPU per box, and NCCL rejects two ranks on one
device, so the NCCL collective itself is covered by the two-GPU test at the end (skipped with
fewer than 2 GPUs); every device kernel of the path is covered here:
  * virtual shards on one GPU: G shards scored separately (fresh index bases), their local keys
    concatenated and merged == tcl_topk of the whole batch, bit-exactly (k = 64, 1024, a shard
    smaller than k, an empty shard);
  * two PROCESSES sharing the GPU (torch.multiprocessing, gloo carrying the keys in place of
    NCCL): each scores its shard through libtcl, exchanges its k keys, merges through libtcl ->
    identical on both ranks and equal to the single-process full-batch top-k.
"""
import os
import socket

import numpy as np
import pytest

import inputs

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2604_12891_b200 import build
    build.build()
    return torch


def _full_topk(torch, m, scores_np, k):
    st = torch.from_numpy(scores_np).cuda()
    idx = torch.empty(k, dtype=torch.int64, device="cuda")
    top = torch.empty(k, dtype=torch.float32, device="cuda")
    m.tcl_topk(st, k, 0, idx, top)
    torch.cuda.synchronize()
    return idx.cpu().numpy(), top.cpu().numpy()


def _virtual_global(torch, m, scores_np, G, k, sizes=None):
    from paper_2604_12891_b200.tcl import shard_range
    n = scores_np.size
    keys = []
    for r in range(G):
        lo, cnt = (sizes[r] if sizes else shard_range(n, G, r))
        kr = torch.empty(k, dtype=torch.int64, device="cuda")
        m.tcl_topk_local_keys(torch.from_numpy(scores_np[lo:lo + cnt].copy()).cuda(), lo, k, kr)
        keys.append(kr)
    cat = torch.cat(keys)
    idx = torch.empty(k, dtype=torch.int64, device="cuda")
    top = torch.empty(k, dtype=torch.float32, device="cuda")
    m.tcl_topk_merge_keys(cat, k, idx, top)
    torch.cuda.synchronize()
    return idx.cpu().numpy(), top.cpu().numpy()


@pytest.mark.parametrize("n,G,k", [(65536, 8, 64), (300000, 4, 1024), (1000, 8, 200), (100, 3, 64)])
def test_virtual_shards_merge_equals_full_topk(torch_cuda, n, G, k):
    from paper_2604_12891_b200 import Model
    c = inputs.config("tiny")
    m = Model(inputs.make_weights(c["dims"], c["seed"]), c["dims"])
    rng = np.random.default_rng(n + G)
    s = np.round(rng.standard_normal(n), 3).astype(np.float32)   # many exact ties across shards
    s[rng.choice(n, max(1, n // 100))] = np.nan
    want = _full_topk(torch_cuda, m, s, k)
    got = _virtual_global(torch_cuda, m, s, G, k)
    assert np.array_equal(got[0], want[0]) and np.array_equal(got[1], want[1])


def test_virtual_shards_small_and_empty(torch_cuda):
    """A shard with n_local < k and an empty shard (its keys are all padding)."""
    from paper_2604_12891_b200 import Model
    c = inputs.config("tiny")
    m = Model(inputs.make_weights(c["dims"], c["seed"]), c["dims"])
    s = np.random.default_rng(7).standard_normal(5000).astype(np.float32)
    sizes = [(0, 10), (10, 0), (10, 4990)]
    got = _virtual_global(torch_cuda, m, s, 3, 64, sizes)
    want = _full_topk(torch_cuda, m, s, 64)
    assert np.array_equal(got[0], want[0]) and np.array_equal(got[1], want[1])
    got = _virtual_global(torch_cuda, m, s[:30].copy(), 2, 64, [(0, 13), (13, 17)])   # k > n: padded
    want = _full_topk(torch_cuda, m, s[:30].copy(), 64)
    assert np.array_equal(got[0], want[0]) and np.array_equal(got[1], want[1])
    assert np.all(got[0][30:] == -1) and np.all(np.isneginf(got[1][30:]))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _proc(rank, world, port, name, n, k, out_q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2604_12891_b200 import Model
    from paper_2604_12891_b200.tcl import shard_range
    c = inputs.config(name)
    d = c["dims"]
    f, l = inputs.make_features(d, n, c["seed"] + 1, workload=name if name in ("tuning", "large") else "tuning")
    lo, cnt = shard_range(n, world, rank)
    m = Model(inputs.make_weights(d, c["seed"]), d)
    sc = torch.empty(cnt, dtype=torch.float32, device="cuda")
    m.tcl_score(torch.from_numpy(f[lo:lo + cnt].copy()).cuda(), torch.from_numpy(l[lo:lo + cnt].copy()).cuda(), sc)
    keys = torch.empty(k, dtype=torch.int64, device="cuda")
    m.tcl_topk_local_keys(sc, lo, k, keys)
    m.tcl_sync_error()
    gathered = [torch.zeros(k, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(gathered, keys.cpu())                      # the exchange (NCCL in tcl_topk_global)
    cat = torch.cat(gathered).cuda()
    idx = torch.empty(k, dtype=torch.int64, device="cuda")
    top = torch.empty(k, dtype=torch.float32, device="cuda")
    m.tcl_topk_merge_keys(cat, k, idx, top)
    torch.cuda.synchronize()
    out_q.put((rank, idx.cpu().numpy().tolist(), top.cpu().numpy().tolist(), sc.cpu().numpy().tolist(), lo))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("name,n,k", [("tuning", 4096, 64), ("large", 3000, 1024), ("tiny", 40, 64)])
def test_two_processes_one_gpu(torch_cuda, name, n, k):
    """World size 2 on one GPU: shard scoring + local keys + exchange + merge through libtcl in two
    processes == the single-process full-batch scores (bit-exact: batch-invariant) and top-k."""
    import torch.multiprocessing as mp
    from paper_2604_12891_b200 import Model
    torch = torch_cuda
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_proc, args=(r, 2, port, name, n, k, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=600) for _ in range(2))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert res[0][1] == res[1][1] and res[0][2] == res[1][2]
    c = inputs.config(name)
    d = c["dims"]
    f, l = inputs.make_features(d, n, c["seed"] + 1, workload=name if name in ("tuning", "large") else "tuning")
    m = Model(inputs.make_weights(d, c["seed"]), d)
    s_full = torch.empty(n, dtype=torch.float32, device="cuda")
    m.tcl_score(torch.from_numpy(f).cuda(), torch.from_numpy(l).cuda(), s_full)
    s_full = s_full.cpu().numpy()
    s_ranks = np.zeros(n, np.float32)
    for _, _, _, s, lo in res:
        s_ranks[lo:lo + len(s)] = s
    assert np.array_equal(s_ranks, s_full)
    wi, wt = _full_topk(torch, m, s_full, k)
    assert np.array_equal(np.array(res[0][1]), wi) and np.array_equal(np.array(res[0][2], np.float32), wt)


_NCCL_SCRIPT = r'''
import os, sys, numpy as np, torch, torch.distributed as dist
sys.path.insert(0, sys.argv[1])
import inputs
from paper_2604_12891_b200 import Model, tcl_comm_unique_id
from paper_2604_12891_b200.tcl import shard_range
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank)
dist.init_process_group("nccl", device_id=torch.device("cuda", rank))
c = inputs.config("large"); d = c["dims"]; n = 20000
f, l = inputs.make_features(d, n, c["seed"] + 1, workload="large")
m = Model(inputs.make_weights(d, c["seed"]), d, device=rank)
obj = [tcl_comm_unique_id() if rank == 0 else None]
dist.broadcast_object_list(obj, src=0)
m.tcl_comm_init(obj[0], world, rank)
lo, cnt = shard_range(n, world, rank)
sc = torch.empty(cnt, device="cuda")
m.tcl_score(torch.from_numpy(f[lo:lo + cnt].copy()).cuda(), torch.from_numpy(l[lo:lo + cnt].copy()).cuda(), sc)
out = []
for k in (64, 1024):
    idx = torch.empty(k, dtype=torch.int64, device="cuda"); top = torch.empty(k, device="cuda")
    m.tcl_topk_global(sc, lo, k, idx, top)
    torch.cuda.synchronize()
    out.append(idx.cpu().numpy())
if rank == 0:
    np.savez(sys.argv[2], k64=out[0], k1024=out[1])
dist.destroy_process_group()
'''


def test_nccl_two_gpus(torch_cuda, tmp_path):
    """tcl_topk_global over a real 2-rank NCCL communicator (needs 2 GPUs; skipped otherwise) ==
    the single-GPU top-k of the whole batch."""
    import subprocess
    import sys
    torch = torch_cuda
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs (gpurun boxes have one)")
    from paper_2604_12891_b200 import Model
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    script = tmp_path / "nccl.py"
    script.write_text(_NCCL_SCRIPT)
    out = tmp_path / "out.npz"
    subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
                    "--master-addr=127.0.0.1", f"--master-port={_free_port()}", str(script), root, str(out)],
                   check=True, timeout=600)
    got = np.load(out)
    c = inputs.config("large")
    d = c["dims"]
    f, l = inputs.make_features(d, 20000, c["seed"] + 1, workload="large")
    m = Model(inputs.make_weights(d, c["seed"]), d)
    s = torch.empty(20000, device="cuda")
    m.tcl_score(torch.from_numpy(f).cuda(), torch.from_numpy(l).cuda(), s)
    s = s.cpu().numpy()
    for k in (64, 1024):
        assert np.array_equal(got[f"k{k}"], _full_topk(torch, m, s, k)[0])
