"""GPU parity of RDU acquisition (tcl_rdu_select).

Primary check: the plain fp64 oracle (oracle.rdu_select_f64 / rdu_follow_f64, two-pass Eq. 3):
every GPU pick must be within a near-tie tolerance of the best fp64 total score given the picks
before it (the R19-style rule for integer decisions taken in floating point).  Secondary check:
the fp32 oracle that evaluates Eqs. 1-3 / line 24 in the kernel's precision and operation order
(reading R21) must give the identical index sequence.
"""
import numpy as np
import pytest

import inputs

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def env():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2604_12891_b200 import Model, build
    build.build()
    c = inputs.config("tiny")
    d = c["dims"]
    return torch, Model(inputs.make_weights(d, c["seed"]), d)


def _gpu_select(torch, m, pool, ops, lab, n_ops, B):
    sel = torch.full((max(B, 1),), -7, dtype=torch.int64, device="cuda")
    ns = torch.full((1,), -1, dtype=torch.int32, device="cuda")
    m.tcl_rdu_select(torch.from_numpy(pool).cuda(), torch.from_numpy(ops).cuda(),
                     torch.from_numpy(lab).cuda(), n_ops, B, sel, ns)
    torch.cuda.synchronize()
    k = int(ns.item())
    return sel[:k].cpu().numpy()


def _case(seed, n, m, n_ops, dist="normal", ties=0):
    rng = np.random.default_rng(seed)
    if dist == "normal":
        pool = rng.normal(size=n).astype(np.float32)
        lab = rng.normal(size=m).astype(np.float32)
    else:   # log-latency-like skewed predictions
        pool = -rng.lognormal(0.0, 1.0, n).astype(np.float32)
        lab = -rng.lognormal(0.0, 1.0, m).astype(np.float32)
    if ties:
        pool = np.round(pool * ties) / ties
        lab = np.round(lab * ties) / ties
    # skewed operator mix (few dominant types, long tail), as in Fig. 4's workload
    p = 1.0 / np.arange(1, n_ops + 1) ** 1.2
    ops = rng.choice(n_ops, n, p=p / p.sum()).astype(np.int32)
    return pool.astype(np.float32), ops, lab.astype(np.float32)


@pytest.mark.parametrize("seed,n,m,n_ops,B,dist,ties", [
    (0, 50, 0, 1, 10, "normal", 0),
    (1, 3000, 100, 5, 200, "normal", 0),
    (2, 4097, 17, 9, 333, "skew", 0),
    (3, 20000, 256, 24, 1000, "skew", 8),     # heavy ties: tie rules decide
    (4, 200000, 1000, 40, 1024, "normal", 0),
    (5, 1000, 10, 3, 1000, "normal", 0),     # budget = pool: shares bind, round ends at the shares
])
def test_rdu_select_parity(env, oracle, seed, n, m, n_ops, B, dist, ties):
    torch, model = env
    pool, ops, lab = _case(seed, n, m, n_ops, dist, ties)
    got = _gpu_select(torch, model, pool, ops, lab, n_ops, B)
    if n * (m + B) <= 3000 * 400:   # fp64 two-pass replay (O(n (m + picks)) per pick)
        near = oracle.rdu_follow_f64(pool, ops, lab, n_ops, B, got, tol=1e-5)
        print(f"seed {seed}: {len(got)} picks, {near} near ties vs fp64")
    want = oracle.rdu_select(pool, ops, lab, n_ops, B)
    assert got.tolist() == want.tolist()


def test_rdu_select_max_pool(env, oracle):
    torch, model = env
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    n = 4096 * sms
    pool, ops, lab = _case(7, n, 40, 16)
    got = _gpu_select(torch, model, pool, ops, lab, 16, 256)
    want = oracle.rdu_select(pool, ops, lab, 16, 256)
    assert got.tolist() == want.tolist()
    from paper_2604_12891_b200.tcl import TclError
    with pytest.raises(TclError):
        _gpu_select(torch, model, np.zeros(n + 1, np.float32), np.zeros(n + 1, np.int32), lab, 16, 4)


def test_rdu_select_edge_cases(env, oracle):
    torch, model = env
    pool = np.float32([0.1, np.nan, 0.9, np.inf, -np.inf, 0.5, 0.7, 0.3])
    ops = np.int32([0, 0, 1, 0, 1, 9, -1, 1])      # 9, -1: outside [0, n_ops) -> never selected
    lab = np.float32([np.nan, 0.2])
    for B in (0, 1, 3, 8):
        got = _gpu_select(torch, model, pool, ops, lab, 2, B)
        assert got.tolist() == oracle.rdu_select(pool, ops, lab, 2, B).tolist()
    flat = np.full(300, 2.5, np.float32)
    got = _gpu_select(torch, model, flat, np.zeros(300, np.int32), np.float32([2.5]), 1, 40)
    assert got.tolist() == list(range(40))


def test_rdu_on_model_predictions(env, oracle):
    """End to end on the rdu configuration: MC-dropout mean predictions of the pool from tcl_score_mc
    (the acquisition input of §8(f)), the first 512 taken as the labeled set."""
    torch, _ = env
    from paper_2604_12891_b200 import Model
    c = inputs.config("rdu")
    d = c["dims"]
    m = Model(inputs.make_weights(d, c["seed"]), d)
    n = 8192
    f, l = inputs.make_features(d, n, c["seed"] + 1, workload="rdu")
    mean = torch.empty(n, device="cuda")
    var = torch.empty(n, device="cuda")
    m.tcl_score_mc(torch.from_numpy(f).cuda(), torch.from_numpy(l).cuda(), c["mc_passes"], 99, 0, mean, var)
    m.tcl_sync_error()
    s = mean.cpu().numpy()
    ops = (np.arange(n) % 13).astype(np.int32)
    pool, lab, pops = s[512:].copy(), s[:512].copy(), ops[512:].copy()
    got = _gpu_select(torch, m, pool, pops, lab, 13, 512)
    assert got.tolist() == oracle.rdu_select(pool, pops, lab, 13, 512).tolist()
    assert len(got) == 512
    # fp64 replay on a 2,000-candidate slice of the same pool
    g2 = _gpu_select(torch, m, pool[:2000].copy(), pops[:2000].copy(), lab[:200].copy(), 13, 200)
    near = oracle.rdu_follow_f64(pool[:2000], pops[:2000], lab[:200], 13, 200, g2, tol=1e-5)
    assert near <= 10
