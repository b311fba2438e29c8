"""GPU parity: the CUDA path (through the C ABI) against the fp64 oracle on the same seeded inputs.

Tolerances (BASELINE.json north_star): |score_gpu - score_ref| <= 1e-4 * max(1, |ref|) for the
fp32 path, <= 2e-2 * max(1, |ref|) for the bf16-projection path (reading R18); top-k indices
bit-exact for the fp32 path (reading R19: exact when no boundary pair is closer than twice the
measured score error; such pairs are listed and counted, not failed).  Invariants (padding,
permutation, batch size, shard) are bit-exact.
"""
import numpy as np
import pytest

import inputs

pytestmark = pytest.mark.gpu

TOL = {inputs.PREC_FP32: 1e-4, inputs.PREC_BF16_PROJ: 2e-2}


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2604_12891_b200 import build
    build.build()
    return torch


def _setup(name, n=None, seed_off=1, dims_over=None, **featkw):
    c = inputs.config(name)
    d = c["dims"] if dims_over is None else c["dims"].replace(**dims_over)
    w = inputs.make_weights(d, c["seed"])
    n = c["n"] if n is None else n
    f, l = inputs.make_features(d, n, c["seed"] + seed_off, workload=featkw.pop("workload", name if name in ("tuning", "rdu", "large", "long") else "tuning"), **featkw)
    return d, w, f, l


def _gpu_score(torch, model, f, l):
    ft = torch.from_numpy(f).cuda()
    lt = torch.from_numpy(l).cuda()
    st = torch.empty(l.shape[0], dtype=torch.float32, device="cuda")
    model.tcl_score(ft, lt, st)
    model.tcl_sync_error()
    return st.cpu().numpy()


def _check_scores(got, ref, prec):
    tol = TOL[prec] * np.maximum(1.0, np.abs(ref))
    err = np.abs(got.astype(np.float64) - ref)
    bad = np.nonzero(err > tol)[0]
    assert bad.size == 0, f"{bad.size} scores out of tolerance; worst {err.max():.3e} at {err.argmax()}"
    return float(err.max())


@pytest.mark.parametrize("name,disc", [("tiny", 0), ("tiny", 1), ("paper", 0), ("tuning", 0)])
def test_score_parity_fp32(torch_cuda, oracle, name, disc):
    from paper_2604_12891_b200 import Model
    d, w, f, l = _setup(name, dims_over=dict(disc=disc))
    m = Model(w, d)
    got = _gpu_score(torch_cuda, m, f, l)
    ref = oracle.score(d, w, f, l)
    err = _check_scores(got, ref, d.precision)
    print(f"{name} disc={disc}: n={len(l)} max|err|={err:.3e} score std={ref.std():.3e}")


@pytest.mark.parametrize("name", ["large", "rdu"])
def test_score_parity_fp32_wide(torch_cuda, oracle, name):
    """The fp32 path (3xTF32 row GEMMs, several N tiles per row, residual epilogue) at d_model 256
    and 128, including MC dropout through the tensor-core epilogue."""
    from paper_2604_12891_b200 import Model
    d, w, f, l = _setup(name, n=300, dims_over=dict(precision=inputs.PREC_FP32))
    m = Model(w, d)
    got = _gpu_score(torch_cuda, m, f, l)
    err = _check_scores(got, oracle.score(d, w, f, l), d.precision)
    mean, var = _mc_gpu(torch_cuda, m, f[:48], l[:48], 3, 17, index_base=2)
    rm, rv = oracle.score_mc(d, w, f[:48], l[:48], 3, 17, index_base=2)
    _check_scores(mean, rm, d.precision)
    assert np.all(np.abs(var - rv) <= 2 * TOL[d.precision] * np.sqrt(np.maximum(rv, 1e-8)) + 1e-7)
    print(f"{name} fp32: max|err|={err:.3e}")


def test_score_parity_bf16_large_small_batch(torch_cuda, oracle):
    from paper_2604_12891_b200 import Model
    d, w, f, l = _setup("large", n=384)
    m = Model(w, d)
    got = _gpu_score(torch_cuda, m, f, l)
    ref = oracle.score(d, w, f, l)
    err = _check_scores(got, ref, d.precision)
    rho = np.corrcoef(np.argsort(np.argsort(got)), np.argsort(np.argsort(ref)))[0, 1]
    print(f"large bf16: max|err|={err:.3e} spearman={rho:.5f}")
    assert rho > 0.99


@pytest.mark.parametrize("name", ["tuning", "rdu", "paper"])
def test_bf16_path_on_fp32_configs(torch_cuda, oracle, name):
    """The d_model-128 configurations run through the bf16-projection path (tcgen05 encoder, in_proj,
    out_proj + LN, fused mixer at d_inner 128, N 8) within that path's 2e-2 bound, MC included."""
    from paper_2604_12891_b200 import Model
    d, w, f, l = _setup(name, n=512)
    d = d.replace(precision=inputs.PREC_BF16_PROJ)
    m = Model(w, d)
    got = _gpu_score(torch_cuda, m, f, l)
    ref = oracle.score(d, w, f, l)
    _check_scores(got, ref, d.precision)
    mean, var = _mc_gpu(torch_cuda, m, f[:64], l[:64], 4, 77, index_base=3)
    rm, rv = oracle.score_mc(d, w, f[:64], l[:64], 4, 77, index_base=3)
    _check_scores(mean, rm, d.precision)


def _rank_metrics(got, ref, k):
    """bf16-path ranking quality against the oracle (reading R18): Spearman rho, top-k overlap, and
    the plain relative error |d| / |ref| (reported: unbounded for scores near 0)."""
    rg = np.argsort(np.argsort(got, kind="stable"), kind="stable")
    rr = np.argsort(np.argsort(ref, kind="stable"), kind="stable")
    rho = float(np.corrcoef(rg, rr)[0, 1])
    k = min(k, len(got))
    ov = len(set(np.argsort(-got, kind="stable")[:k]) & set(np.argsort(-ref, kind="stable")[:k]))
    rel = np.abs(got - ref) / np.maximum(np.abs(ref), 1e-30)
    return rho, ov, float(np.median(rel)), float(np.percentile(rel, 99))


@pytest.mark.parametrize("variant", ["default", "stress", "full_length"])
def test_bf16_large_input_variants(torch_cuda, oracle, variant):
    """SURVEY §8(d) input variants at the `large` model: the Tenset-style default, the stress
    variant (iid N(0,1) real slots) and the full-length variant (T = L), 1,024 candidates each:
    R18 bound, Spearman rho >= 0.999 and top-64 overlap >= 60 / 64 against the fp64 oracle."""
    from paper_2604_12891_b200 import Model
    kw = {"default": {}, "stress": {"stress": True}, "full_length": {"full_length": True}}[variant]
    d, w, f, l = _setup("large", n=1024, **kw)
    m = Model(w, d)
    got = _gpu_score(torch_cuda, m, f, l)
    ref = oracle.score(d, w, f, l)
    err = _check_scores(got, ref, d.precision)
    rho, ov, rel50, rel99 = _rank_metrics(got, ref, 64)
    print(f"large bf16 {variant}: max|d|={err:.3e} score std={ref.std():.3e} max|d|/std={err / ref.std():.3f} "
          f"rel median={rel50:.2e} p99={rel99:.2e} spearman={rho:.6f} top64 overlap={ov}/64")
    assert rho >= 0.999 and ov >= 60


@pytest.mark.parametrize("name,disc", [("tiny", 0), ("tiny", 1), ("large", 1), ("tuning", 1)])
def test_bf16_small_dmodel_and_euler(torch_cuda, oracle, name, disc):
    """bf16 path at d_model 64 (tiny: the in-kernel residual + LayerNorm epilogue of k_gemm_tc
    (EPI 3) and the d_inner-64 mixer) and with Euler-B discretisation (DISC 1 scan branch)."""
    from paper_2604_12891_b200 import Model
    d, w, f, l = _setup(name, n=512, dims_over=dict(disc=disc, precision=inputs.PREC_BF16_PROJ))
    m = Model(w, d)
    got = _gpu_score(torch_cuda, m, f, l)
    ref = oracle.score(d, w, f, l)
    err = _check_scores(got, ref, d.precision)
    rho, ov, _, _ = _rank_metrics(got, ref, 16)
    print(f"{name} bf16 disc={disc}: max|d|={err:.3e} std={ref.std():.3e} spearman={rho:.6f} top16={ov}/16")
    assert rho >= 0.999 and ov >= 14
    # batch invariance on this instantiation too
    assert np.array_equal(_gpu_score(torch_cuda, m, f[100:300], l[100:300]), got[100:300])


def test_full_size_sampled_parity_large(torch_cuda, oracle):
    """BASELINE.json full size (65,536 candidates, the bench configuration); the oracle scores a
    sample of candidates one by one, plus every top-k member."""
    from paper_2604_12891_b200 import Model
    c = inputs.config("large")
    d, w, f, l = _setup("large")
    m = Model(w, d)
    got = _gpu_score(torch_cuda, m, f, l)
    assert np.isfinite(got).all()
    rng = np.random.default_rng(0)
    sample = np.unique(np.concatenate([rng.choice(len(l), 48, replace=False),
                                       np.argsort(-got, kind="stable")[:c["topk"]][:16]]))
    ref = oracle.score(d, w, f[sample], l[sample])
    err = _check_scores(got[sample], ref, d.precision)
    rel = np.abs(got[sample] - ref) / np.maximum(np.abs(ref), 1e-30)
    print(f"large full size: sampled max|d|={err:.3e} rel median={np.median(rel):.2e}")


def test_full_size_sampled_parity_rdu_mc(torch_cuda, oracle):
    """BASELINE.json "RDU uncertainty" at full size: 16,384 candidates x 10 MC-dropout passes in one
    tcl_score_mc call (the masks are keyed by global index, so a sampled candidate i is re-scored by
    the oracle alone with index_base = i)."""
    from paper_2604_12891_b200 import Model
    c = inputs.config("rdu")
    d, w, f, l = _setup("rdu")
    assert len(l) == c["n"] == 16384
    m = Model(w, d)
    mean, var = _mc_gpu(torch_cuda, m, f, l, c["mc_passes"], 4321, index_base=0)
    assert np.isfinite(mean).all() and (var >= 0).all()
    rng = np.random.default_rng(1)
    for i in rng.choice(len(l), 24, replace=False):
        rm, rv = oracle.score_mc(d, w, f[i:i + 1], l[i:i + 1], c["mc_passes"], 4321, index_base=int(i))
        _check_scores(mean[i:i + 1], rm, d.precision)
        assert abs(var[i] - rv[0]) <= 2 * TOL[d.precision] * np.sqrt(max(rv[0], 1e-8)) + 1e-7


def test_sampled_parity_long_131072(torch_cuda, oracle):
    """BASELINE.json "long-range" at its per-GPU share on 8 GPUs (1,048,576 / 8 = 131,072 candidates,
    L = 128): sampled candidates and the head of the top-k against the oracle."""
    from paper_2604_12891_b200 import Model
    d, w, f, l = _setup("long", n=131072)
    m = Model(w, d)
    got = _gpu_score(torch_cuda, m, f, l)
    assert np.isfinite(got).all()
    rng = np.random.default_rng(2)
    sample = np.unique(np.concatenate([rng.choice(len(l), 12, replace=False),
                                       np.argsort(-got, kind="stable")[:4]]))
    ref = oracle.score(d, w, f[sample], l[sample])
    _check_scores(got[sample], ref, d.precision)


def test_padding_invariance_bitexact(torch_cuda):
    from paper_2604_12891_b200 import Model
    d, w, f, l = _setup("tiny")
    m = Model(w, d)
    s0 = _gpu_score(torch_cuda, m, f, l)
    for pad in ("random", np.nan, np.inf):
        _, _, f2, l2 = _setup("tiny", pad_value=pad)
        assert np.array_equal(l2, l)
        assert np.array_equal(_gpu_score(torch_cuda, m, f2, l2), s0), pad


@pytest.mark.parametrize("name", ["tiny", "large"])
def test_permutation_and_batch_invariance_bitexact(torch_cuda, name):
    from paper_2604_12891_b200 import Model
    d, w, f, l = _setup(name, n=1000)
    m = Model(w, d)
    s = _gpu_score(torch_cuda, m, f, l)
    perm = np.random.default_rng(3).permutation(len(l))
    assert np.array_equal(_gpu_score(torch_cuda, m, f[perm], l[perm]), s[perm])
    assert np.array_equal(_gpu_score(torch_cuda, m, f[:37], l[:37]), s[:37])
    assert np.array_equal(_gpu_score(torch_cuda, m, f[500:501], l[500:501]), s[500:501])
    # shard invariance: a fresh model (fresh workspace) on a shard
    m2 = Model(w, d)
    assert np.array_equal(_gpu_score(torch_cuda, m2, f[250:750], l[250:750]), s[250:750])


def test_scan_work_assignment_bitexact(torch_cuda):
    """k_scan claims groups of 8 candidates dynamically at large batches (>= 4 groups per CTA) and
    keeps the static row partition below: a 16,000-candidate batch (dynamic) and its 500-candidate
    slices (static) score every candidate bit-identically, as does the batch permuted."""
    from paper_2604_12891_b200 import Model
    d, w, f, l = _setup("large", n=16000)
    m = Model(w, d)
    s = _gpu_score(torch_cuda, m, f, l)
    for a in (0, 7777, 15500):
        assert np.array_equal(_gpu_score(torch_cuda, m, f[a:a + 500], l[a:a + 500]), s[a:a + 500])
    perm = np.random.default_rng(5).permutation(len(l))
    assert np.array_equal(_gpu_score(torch_cuda, m, f[perm], l[perm]), s[perm])


@pytest.mark.parametrize("name,prec", [("tuning", inputs.PREC_FP32), ("large", inputs.PREC_BF16_PROJ)])
def test_head_forms_bitexact(torch_cuda, name, prec):
    """The one-launch head (batches < 8,192) and the five-launch head (larger batches) compute each
    candidate identically: a 9,000-candidate batch and its 300-candidate slice agree bit for bit."""
    from paper_2604_12891_b200 import Model
    d, w, f, l = _setup(name, n=9000, dims_over=dict(precision=prec))
    m = Model(w, d)
    s = _gpu_score(torch_cuda, m, f, l)
    assert np.array_equal(_gpu_score(torch_cuda, m, f[4000:4300], l[4000:4300]), s[4000:4300])


def test_edge_lengths_and_invalid(torch_cuda, oracle):
    from paper_2604_12891_b200 import Model, TclError
    d, w, f, l = _setup("tiny", n=64)
    l = l.copy()
    l[:8] = 1                      # shortest
    l[8:16] = d.max_len            # longest
    m = Model(w, d)
    got = _gpu_score(torch_cuda, m, f, l)
    _check_scores(got, oracle.score(d, w, f, l), d.precision)
    l[3] = 0
    l[9] = d.max_len + 1
    torch = torch_cuda
    st = torch.empty(64, dtype=torch.float32, device="cuda")
    m.tcl_score(torch.from_numpy(f).cuda(), torch.from_numpy(l).cuda(), st)
    with pytest.raises(TclError) as e:
        m.tcl_sync_error()
    assert e.value.code == -3       # TCL_ELEN
    s = st.cpu().numpy()
    assert np.isnan(s[3]) and np.isnan(s[9])
    ok = np.ones(64, bool)
    ok[[3, 9]] = False
    assert np.array_equal(s[ok], got[ok])   # other candidates unaffected, bit-exact
    m.tcl_sync_error()                       # the flag was cleared


def test_empty_batch_is_noop(torch_cuda):
    from paper_2604_12891_b200 import Model
    torch = torch_cuda
    d, w, f, l = _setup("tiny", n=4)
    m = Model(w, d)
    e = torch.empty(0, dtype=torch.float32, device="cuda")
    m.tcl_score(e, torch.empty(0, dtype=torch.int32, device="cuda"), e)
    m.tcl_sync_error()


# ------------------------------------------------------------------------------------ top-k
def _topk_gpu(torch, m, s, k, index_base=0):
    st = torch.from_numpy(s).cuda()
    idx = torch.empty(k, dtype=torch.int64, device="cuda")
    top = torch.empty(k, dtype=torch.float32, device="cuda")
    m.tcl_topk(st, k, index_base, idx, top)
    torch.cuda.synchronize()
    return idx.cpu().numpy(), top.cpu().numpy()


@pytest.mark.parametrize("n,k", [(1, 1), (100, 16), (8192, 64), (8193, 64), (65536, 64),
                                 (300000, 1024), (50, 64), (20000, 4096),
                                 (8192, 256), (100000, 256), (100000, 257), (1000000, 64),
                                 # the radix-select / bitonic-tournament boundary (k <= 1024 radix)
                                 (100000, 1024), (100000, 1025), (700, 1000), (300, 257)])
def test_topk_bitexact_vs_stable_sort(torch_cuda, n, k):
    from paper_2604_12891_b200 import Model
    d, w, _, _ = _setup("tiny", n=2)
    m = Model(w, d)
    rng = np.random.default_rng(n + k)
    s = np.round(rng.standard_normal(n), 3).astype(np.float32)   # many exact ties
    s[rng.choice(n, max(1, n // 100))] = np.nan
    if n > 5:
        s[2] = -0.0
        s[4] = 0.0
    idx, top = _topk_gpu(torch_cuda, m, s, k, index_base=7)
    key = np.where(np.isnan(s), -np.inf, s).astype(np.float64)
    key[key == 0] = 0.0
    order = np.lexsort((np.arange(n), -key))[:min(k, n)]
    assert np.array_equal(idx[:len(order)], order + 7)
    assert np.array_equal(top[:len(order)].astype(np.float64), key[order])
    if k > n:
        assert np.all(idx[n:] == -1) and np.all(np.isneginf(top[n:]))


def test_topk_matches_oracle_fp32(torch_cuda, oracle):
    """TK1: GPU top-k of the GPU scores == oracle top-k of the same scores.
    TK2: == oracle top-k of the oracle scores, except pairs closer than 2x the score error."""
    from paper_2604_12891_b200 import Model
    c = inputs.config("tuning")
    d, w, f, l = _setup("tuning")
    m = Model(w, d)
    got = _gpu_score(torch_cuda, m, f, l)
    k = c["topk"]
    gi, gt = _topk_gpu(torch_cuda, m, got, k)
    oi, ot = oracle.topk(got, k)
    assert np.array_equal(gi, oi) and np.array_equal(gt, ot)
    ref = oracle.score(d, w, f, l)
    ri, _ = oracle.topk(ref, k)
    err = np.abs(got - ref).max()
    srt = np.sort(ref)[::-1]
    gaps = np.abs(np.diff(srt[:k + 1]))
    # exact duplicates (identical candidates) tie identically on both sides (batch-invariant scores,
    # index tie-break), so only distinct values closer than twice the error are ambiguous
    close = np.sum((gaps > 0) & (gaps <= 2 * err))
    if close == 0:
        assert np.array_equal(gi, ri)
    else:
        print(f"TK2: {close} ambiguous adjacent pairs within 2*err={2 * err:.2e}; "
              f"overlap {len(set(gi) & set(ri))}/{k}")
        assert len(set(gi) & set(ri)) >= k - close


def test_topk_global_single_rank(torch_cuda):
    """NCCL path with one rank == local top-k (the multi-rank merge is the same kernel)."""
    from paper_2604_12891_b200 import Model, tcl_comm_unique_id
    torch = torch_cuda
    d, w, _, _ = _setup("tiny", n=2)
    m = Model(w, d)
    m.tcl_comm_init(tcl_comm_unique_id(), 1, 0)
    s = np.random.default_rng(1).standard_normal(30000).astype(np.float32)
    li, lt = _topk_gpu(torch, m, s, 64, index_base=1000)
    st = torch.from_numpy(s).cuda()
    gi = torch.empty(64, dtype=torch.int64, device="cuda")
    gt = torch.empty(64, dtype=torch.float32, device="cuda")
    m.tcl_topk_global(st, 1000, 64, gi, gt)
    torch.cuda.synchronize()
    assert np.array_equal(gi.cpu().numpy(), li) and np.array_equal(gt.cpu().numpy(), lt)


# ------------------------------------------------------------------------------------ MC
def _mc_gpu(torch, m, f, l, passes, seed, index_base=0):
    n = len(l)
    mean = torch.empty(n, dtype=torch.float32, device="cuda")
    var = torch.empty(n, dtype=torch.float32, device="cuda")
    m.tcl_score_mc(torch.from_numpy(f).cuda(), torch.from_numpy(l).cuda(), passes, seed, index_base, mean, var)
    m.tcl_sync_error()
    return mean.cpu().numpy(), var.cpu().numpy()


def test_mc_p0_equals_score_bitexact(torch_cuda):
    from paper_2604_12891_b200 import Model
    d, w, f, l = _setup("tiny", dims_over=dict(dropout_p=0.0))
    m = Model(w, d)
    s = _gpu_score(torch_cuda, m, f, l)
    mean, var = _mc_gpu(torch_cuda, m, f, l, 3, 5)
    assert np.array_equal(mean, s) and np.all(var == 0)


@pytest.mark.parametrize("name", ["tiny", "rdu"])
def test_mc_parity(torch_cuda, oracle, name):
    from paper_2604_12891_b200 import Model
    c = inputs.config(name)
    d, w, f, l = _setup(name, n=256)
    passes = c["mc_passes"] or 4
    m = Model(w, d)
    mean, var = _mc_gpu(torch_cuda, m, f, l, passes, 1234, index_base=77)
    rm, rv = oracle.score_mc(d, w, f, l, passes, 1234, index_base=77)
    _check_scores(mean, rm, d.precision)
    # variance: absolute tolerance scaled by the score tolerance (var = E[(s - mean)^2])
    assert np.all(np.abs(var - rv) <= 2 * TOL[d.precision] * np.sqrt(np.maximum(rv, 1e-8)) + 1e-7)
    # shard invariance of the masks (keyed by global index)
    m2, v2 = _mc_gpu(torch_cuda, m, f[100:], l[100:], passes, 1234, index_base=177)
    assert np.array_equal(m2, mean[100:]) and np.array_equal(v2, var[100:])


def test_mc_batched_passes_across_chunks(torch_cuda, oracle):
    """tcl_score_mc runs its passes batched (passes x nc virtual candidates per forward, nc =
    chunk capacity / passes = 16,777 at rdu's max_len 25): 20,000 candidates x 10 passes take two
    chunks.  A slice straddling the chunk seam is bit-identical to the full batch (masks keyed by
    (pass, global index)), and sampled candidates on both sides match the oracle."""
    from paper_2604_12891_b200 import Model
    c = inputs.config("rdu")
    d, w, f, l = _setup("rdu", n=20000)
    passes = c["mc_passes"]
    m = Model(w, d)
    mean, var = _mc_gpu(torch_cuda, m, f, l, passes, 99, index_base=5)
    m2, v2 = _mc_gpu(torch_cuda, m, f[16000:17600], l[16000:17600], passes, 99, index_base=16005)
    assert np.array_equal(m2, mean[16000:17600]) and np.array_equal(v2, var[16000:17600])
    sample = np.array([0, 1, 16775, 16776, 16777, 16778, 19999])
    rm = np.empty(sample.size); rv = np.empty(sample.size)
    for j, i in enumerate(sample):   # the oracle keys masks by index_base + position: one call each
        a, b = oracle.score_mc(d, w, f[i:i + 1], l[i:i + 1], passes, 99, index_base=5 + int(i))
        rm[j], rv[j] = a[0], b[0]
    _check_scores(mean[sample], rm, d.precision)
    assert np.all(np.abs(var[sample] - rv) <= 2 * TOL[d.precision] * np.sqrt(np.maximum(rv, 1e-8)) + 1e-7)


# ------------------------------------------------------------------------------------ host e2e
@pytest.mark.parametrize("n", [1000, 20000, 70000])
def test_score_host_matches_device(torch_cuda, n):
    """tcl_score_host (pinned host buffers, pipelined sub-chunks: one for n <= 16,384, else
    4,096, 16,384, ...) is bit-identical to tcl_score on device-resident inputs."""
    from paper_2604_12891_b200 import Model
    d, w, f, l = _setup("tuning", n=n)
    m = Model(w, d)
    s_dev = _gpu_score(torch_cuda, m, f, l)
    s_host, idx, top = m.tcl_score_host(f, l, k=64)
    assert np.array_equal(s_host, s_dev)
    gi, gt = _topk_gpu(torch_cuda, m, s_dev, 64)
    assert np.array_equal(idx, gi) and np.array_equal(top, gt)


# ------------------------------------------------------------------------------------ bf16 path extras
def test_bf16_mc_parity(torch_cuda, oracle):
    """MC dropout through the tcgen05 epilogues (Philox masks at enc h1/h2) and the decoder."""
    from paper_2604_12891_b200 import Model
    d, w, f, l = _setup("large", n=48)
    m = Model(w, d)
    mean, var = _mc_gpu(torch_cuda, m, f, l, 3, 99, index_base=5)
    rm, rv = oracle.score_mc(d, w, f, l, 3, 99, index_base=5)
    _check_scores(mean, rm, d.precision)
    assert np.all(np.abs(var - rv) <= 2 * TOL[d.precision] * np.sqrt(np.maximum(rv, 1e-8)) + 1e-5)
    s = _gpu_score(torch_cuda, Model(w, d.replace(dropout_p=0.0)), f, l)
    m0 = Model(w, d.replace(dropout_p=0.0))
    mean0, var0 = _mc_gpu(torch_cuda, m0, f, l, 2, 99)
    assert np.array_equal(mean0, s) and np.all(var0 == 0)


def test_bf16_invalid_lengths_and_host_path(torch_cuda, oracle):
    from paper_2604_12891_b200 import Model, TclError
    d, w, f, l = _setup("large", n=40)
    l = l.copy()
    l[:4] = 1
    l[4:8] = d.max_len
    m = Model(w, d)
    good = _gpu_score(torch_cuda, m, f, l)
    _check_scores(good, oracle.score(d, w, f, l), d.precision)
    s_host, idx, top = m.tcl_score_host(f, l, k=8)
    assert np.array_equal(s_host, good)
    l2 = l.copy()
    l2[10] = 0
    torch = torch_cuda
    st = torch.empty(40, dtype=torch.float32, device="cuda")
    m.tcl_score(torch.from_numpy(f).cuda(), torch.from_numpy(l2).cuda(), st)
    with pytest.raises(TclError):
        m.tcl_sync_error()
    s2 = st.cpu().numpy()
    ok = np.arange(40) != 10
    assert np.isnan(s2[10]) and np.array_equal(s2[ok], good[ok])


@pytest.mark.parametrize("name", ["tuning", "large"])
def test_mc_batched_invalid_lengths_and_one_pass(torch_cuda, name):
    """Batched MC passes with invalid lengths in the batch: those candidates get NaN mean and var
    (and TCL_ELEN), every other candidate is bit-identical to the same batch with valid lengths
    there (masks keyed by (pass, global index)); one pass: var == 0 exactly."""
    from paper_2604_12891_b200 import Model, TclError
    torch = torch_cuda
    d, w, f, l = _setup(name, n=50)
    m = Model(w, d)
    mean, var = _mc_gpu(torch, m, f, l, 4, 31, index_base=9)
    l2 = l.copy()
    l2[[0, 17, 49]] = [0, d.max_len + 1, -3]
    mt, vt = torch.empty(50, device="cuda"), torch.empty(50, device="cuda")
    m.tcl_score_mc(torch.from_numpy(f).cuda(), torch.from_numpy(l2).cuda(), 4, 31, 9, mt, vt)
    with pytest.raises(TclError):
        m.tcl_sync_error()
    m2, v2 = mt.cpu().numpy(), vt.cpu().numpy()
    bad = np.zeros(50, bool)
    bad[[0, 17, 49]] = True
    assert np.all(np.isnan(m2[bad])) and np.all(np.isnan(v2[bad]))
    assert np.array_equal(m2[~bad], mean[~bad]) and np.array_equal(v2[~bad], var[~bad])
    m1, v1 = _mc_gpu(torch, m, f, l, 1, 31, index_base=9)
    assert np.all(v1 == 0) and np.all(np.isfinite(m1))


def test_bf16_long_config_small_batch(torch_cuda, oracle):
    """`long` model (L = 128) on a small batch: parity + batch invariance across chunks."""
    from paper_2604_12891_b200 import Model
    d, w, f, l = _setup("long", n=64)
    m = Model(w, d)
    got = _gpu_score(torch_cuda, m, f, l)
    _check_scores(got, oracle.score(d, w, f, l), d.precision)


# ------------------------------------------------------------------------------------ CUDA graphs
@pytest.mark.parametrize("name,prec", [("tiny", inputs.PREC_FP32), ("tiny", inputs.PREC_BF16_PROJ),
                                       ("paper", inputs.PREC_FP32), ("large", inputs.PREC_BF16_PROJ)])
def test_graph_replay_bitexact(torch_cuda, name, prec):
    """TCL_OPT_GRAPHS: the 1st call launches directly, the 2nd is captured and launched, later ones
    replay -- every one bit-identical to a model that always launches directly (score, MC, top-k),
    including after the workspace grew (the graphs that baked in the old buffers are dropped)."""
    from paper_2604_12891_b200 import Model
    torch = torch_cuda
    d, w, f, l = _setup(name, n=300, dims_over=dict(precision=prec))
    g = Model(w, d)
    ref = Model(w, d)
    ref.use_graphs(False)
    ft, lt = torch.from_numpy(f).cuda(), torch.from_numpy(l).cuda()
    want = _gpu_score(torch, ref, f, l)
    s = torch.empty(300, device="cuda")
    n0 = g.launch_count()
    for it in range(4):
        s.fill_(float("nan"))
        g.tcl_score(ft, lt, s)
        g.tcl_sync_error()
        assert np.array_equal(s.cpu().numpy(), want), it
    per_call = (g.launch_count() - n0) / 4
    assert per_call == (ref.launch_count()), (per_call, ref.launch_count())
    wm, wv = _mc_gpu(torch, ref, f, l, 3, 9, index_base=11)
    for it in range(3):
        mm, vv = _mc_gpu(torch, g, f, l, 3, 9, index_base=11)
        assert np.array_equal(mm, wm) and np.array_equal(vv, wv), it
    wi, wt = _topk_gpu(torch, ref, want, 16, index_base=5)
    for it in range(3):
        gi, gt = _topk_gpu(torch, g, want, 16, index_base=5)
        assert np.array_equal(gi, wi) and np.array_equal(gt, wt), it
    # a larger batch reallocates the workspace: the old graphs must not be replayed
    _, _, f2, l2 = _setup(name, n=900, dims_over=dict(precision=prec), seed_off=4)
    want2 = _gpu_score(torch, ref, f2, l2)
    for it in range(3):
        assert np.array_equal(_gpu_score(torch, g, f2, l2), want2), it
    s.fill_(float("nan"))
    g.tcl_score(ft, lt, s)
    assert np.array_equal(s.cpu().numpy(), want)


# ------------------------------------------------------------------------------------ chunked scan
@pytest.mark.parametrize("name,disc", [("tiny", 0), ("tiny", 1), ("paper", 0), ("tuning", 0), ("rdu", 1)])
def test_chunked_scan_parity_and_invariance(torch_cuda, oracle, name, disc):
    """TCL_OPT_SCAN = chunked: the fp32 mixer with the warp-shuffle chunked scan across L (one CTA
    per candidate, lanes = tokens, associative (a, b) operator) within the fp32 bound of the oracle,
    within 2e-6 of the sequential scan, and bit-exact under permutation / batch size / sharding."""
    from paper_2604_12891_b200 import Model
    d, w, f, l = _setup(name, n=700, dims_over=dict(disc=disc))
    l = l.copy()
    l[:5] = 1
    l[5:10] = d.max_len
    m = Model(w, d)
    m.scan_mode("chunked")
    got = _gpu_score(torch_cuda, m, f, l)
    ref = oracle.score(d, w, f, l)
    err = _check_scores(got, ref, d.precision)
    seq = Model(w, d)
    seq.scan_mode("sequential")
    s_seq = _gpu_score(torch_cuda, seq, f, l)
    assert np.abs(got - s_seq).max() <= 2e-6 * max(1.0, np.abs(s_seq).max())
    perm = np.random.default_rng(5).permutation(len(l))
    assert np.array_equal(_gpu_score(torch_cuda, m, f[perm], l[perm]), got[perm])
    assert np.array_equal(_gpu_score(torch_cuda, m, f[123:124], l[123:124]), got[123:124])
    m2 = Model(w, d)
    m2.scan_mode("chunked")
    assert np.array_equal(_gpu_score(torch_cuda, m2, f[300:650], l[300:650]), got[300:650])
    print(f"{name} disc={disc} chunked: max|err|={err:.3e} vs sequential {np.abs(got - s_seq).max():.2e}")


# Non-default dimensions: the templated kernels' other instantiations (d_inner != d_model through
# expand 2, d_state 8, other dt_ranks), on both precision paths.  Each case runs the full model
# against the oracle; the bf16 path also checks the ranking (reading R18).
@pytest.mark.parametrize("base,over", [
    ("tuning", dict(expand=2)),                  # d_model 128 -> d_inner 256 (N 8): k_inconv 2-CTA split, K = 128
    ("tiny", dict(expand=2)),                    # d_model 64 -> d_inner 128 (N 16)
    ("large", dict(n_layer=1, d_state=8)),       # d_inner 256 with N 8: 8-float B / C, k_xdt's NXP 32
    ("large", dict(n_layer=2, dt_rank=8)),       # dt_r narrower than ceil(d_model / 16)
    ("tuning", dict(d_state=16, dt_rank=4)),     # d_model 128 with N 16 and dt_rank 4
])
@pytest.mark.parametrize("prec", [inputs.PREC_FP32, inputs.PREC_BF16_PROJ])
def test_score_parity_other_dims(torch_cuda, oracle, base, over, prec):
    from paper_2604_12891_b200 import Model
    d, w, f, l = _setup(base, n=400, dims_over=dict(over, precision=prec), workload="large")
    m = Model(w, d)
    got = _gpu_score(torch_cuda, m, f, l)
    ref = oracle.score(d, w, f, l)
    err = _check_scores(got, ref, d.precision)
    msg = f"{base} {over} prec {prec}: max|err|={err:.3e} std={ref.std():.3e}"
    if prec == inputs.PREC_BF16_PROJ:
        from scipy.stats import spearmanr
        rho = spearmanr(got, ref).correlation
        assert rho >= 0.999, f"spearman {rho:.5f}"
        msg += f" spearman={rho:.6f}"
    print(msg)


def test_score_parity_fp32_tf32_bn32_kb8(torch_cuda, oracle):
    """Encoder widths (256, 96): linear 2 has N = 96 (32-column 3xTF32 tiles) and K = 256 (8 K-blocks),
    the (bn 32, kb 8) instantiation (missing from the dispatcher before: a silent no-op launch)."""
    from paper_2604_12891_b200 import Model
    d, w, f, l = _setup("tuning", n=200, dims_over=dict(n_layer=1, enc_dims=(256, 96, 128), precision=inputs.PREC_FP32))
    m = Model(w, d)
    got = _gpu_score(torch_cuda, m, f, l)
    _check_scores(got, oracle.score(d, w, f, l), d.precision)


def test_reserve_then_score_and_mc(torch_cuda):
    """tcl_reserve(n_max, mc_passes_max) pre-allocates for batched MC passes; results equal an
    unreserved model bit for bit; an oversized n_max reserves the whole arena without overflow."""
    from paper_2604_12891_b200 import Model
    d, w, f, l = _setup("tuning", n=700)
    m0 = Model(w, d)
    mean0, var0 = _mc_gpu(torch_cuda, m0, f, l, 5, 11, index_base=3)
    s0 = _gpu_score(torch_cuda, m0, f, l)
    m = Model(w, d)
    m.reserve(700, 5)
    mean, var = _mc_gpu(torch_cuda, m, f, l, 5, 11, index_base=3)
    assert np.array_equal(mean, mean0) and np.array_equal(var, var0)
    assert np.array_equal(_gpu_score(torch_cuda, m, f, l), s0)
    m2 = Model(w, d)
    m2.reserve(1 << 40, 1 << 20)
    assert np.array_equal(_gpu_score(torch_cuda, m2, f, l), s0)
