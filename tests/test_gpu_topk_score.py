"""GPU parity of the Top-k score (tcl_topk_score, Eq. 12) against oracle.topk_score.

Ranking is integer work (exact), the per-task terms are exact fp64 products, so only the order of
the fp64 sums differs: the scores must agree to 1e-12 relative; repeated calls are bit-identical.
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


def _gpu(torch, m, sc, lat, off, w, ks, max_len=None):
    res = torch.empty(3 * len(ks), dtype=torch.float64, device="cuda")
    ml = int(np.diff(off).max()) if max_len is None else max_len
    m.tcl_topk_score(torch.from_numpy(sc).cuda(), torch.from_numpy(lat).cuda(), torch.from_numpy(off).cuda(),
                     torch.from_numpy(w).cuda(), ml, ks, res)
    torch.cuda.synchronize()
    r = res.cpu().numpy()
    return r[:len(ks)], r[len(ks):2 * len(ks)], r[2 * len(ks):]


@pytest.mark.parametrize("n_tasks,min_len,max_len,tq", [(1, 3, 3, 0.0), (100, 16, 400, 0.0),
                                                         (500, 16, 4096, 0.0), (300, 1, 700, 0.5),
                                                         (7, 9000, 16384, 0.0)])
def test_topk_score_parity(env, oracle, n_tasks, min_len, max_len, tq):
    torch, m = env
    sc, lat, off, w = inputs.make_eval_tasks(n_tasks, 17 + n_tasks, min_len=min_len, max_len=max_len, tie_quant=tq)
    sc[::53] = np.nan
    ks = [1, 5, 10, 64, 100000]
    got, gn, gd = _gpu(torch, m, sc, lat, off, w, ks)
    want, wn, wd = oracle.topk_score(sc, lat, off, w, ks)
    np.testing.assert_allclose(got, want, rtol=1e-12)
    np.testing.assert_allclose(gn, wn, rtol=1e-12)
    np.testing.assert_allclose(gd, wd, rtol=1e-12)
    again = _gpu(torch, m, sc, lat, off, w, ks)[0]
    assert np.array_equal(again, got)


def test_topk_score_spec_example_and_errors(env):
    torch, m = env
    got = _gpu(torch, m, np.float32([0.1, 0.2, 0.9]), np.float32([2, 4, 8]), np.int64([0, 3]), np.float32([1]), [1, 2, 3])[0]
    assert got.tolist() == [0.25, 0.5, 1.0]
    from paper_2604_12891_b200.tcl import TclError
    sc, lat, off, w = inputs.make_eval_tasks(10, 2, max_len=64)
    _gpu(torch, m, sc, lat, off, w, [1], max_len=int(np.diff(off).max()) - 1)   # a task exceeds the cap
    with pytest.raises(TclError):
        m.tcl_sync_error()
    m.tcl_sync_error()   # sticky flag cleared by the read
    with pytest.raises(TclError):
        _gpu(torch, m, sc, lat, off, w, [0])


def test_topk_score_on_model_predictions(env, oracle):
    """Eq. 12 over the tuning model's own predictions: 64 tasks of 64 candidates each."""
    torch, _ = env
    from paper_2604_12891_b200 import Model
    c = inputs.config("tuning")
    d = c["dims"]
    model = Model(inputs.make_weights(d, c["seed"]), d)
    f, l = inputs.make_features(d, 4096, c["seed"] + 1, workload="tuning")
    s = torch.empty(4096, device="cuda")
    model.tcl_score(torch.from_numpy(f).cuda(), torch.from_numpy(l).cuda(), s)
    model.tcl_sync_error()
    sc = s.cpu().numpy()
    rng = np.random.default_rng(0)
    lat = np.exp(rng.normal(-6, 1, 4096)).astype(np.float32)
    off = np.arange(0, 4097, 64, dtype=np.int64)
    w = rng.integers(1, 9, 64).astype(np.float32)
    got = _gpu(torch, model, sc, lat, off, w, [1, 5])[0]
    want = oracle.topk_score(sc, lat, off, w, [1, 5])[0]
    np.testing.assert_allclose(got, want, rtol=1e-12)
