"""Pins of the Top-k score oracle (Eq. 12, §7.1.2; reading R22).

Fixed against: SPEC's worked example, the closed forms of a perfect and a reversed predictor,
k >= task size, weight-scale invariance, monotonicity in k, and an fp64 brute force written
independently with numpy's lexsort.
"""
import numpy as np
import pytest

import inputs


def test_spec_example(oracle):
    # SPEC evalkit.topk_score: one task, latencies [2, 4, 8], the 8-latency program ranked first -> 2/8
    out, num, den = oracle.topk_score([0.1, 0.2, 0.9], [2, 4, 8], [0, 3], [1], [1])
    assert out[0] == 0.25 and num[0] == 2.0 and den[0] == 8.0


def test_perfect_predictor_is_one(oracle):
    sc, lat, off, w = inputs.make_eval_tasks(40, 3, max_len=300)
    out, _, _ = oracle.topk_score(-np.log(lat), lat, off, w, [1, 5, 10])
    np.testing.assert_array_equal(out, 1.0)


def test_reversed_predictor_closed_form(oracle):
    sc, lat, off, w = inputs.make_eval_tasks(30, 4, max_len=200)
    out, _, _ = oracle.topk_score(lat, lat, off, w, [1])   # worst first: Top-1 = sum min w / sum max w
    mins = np.array([lat[off[t]:off[t + 1]].min() for t in range(30)], np.float64)
    maxs = np.array([lat[off[t]:off[t + 1]].max() for t in range(30)], np.float64)
    assert out[0] == pytest.approx((mins * w).sum() / (maxs * w).sum(), rel=1e-14)


def test_k_beyond_task_size_and_monotone(oracle):
    sc, lat, off, w = inputs.make_eval_tasks(25, 5, max_len=100)
    out, _, _ = oracle.topk_score(sc, lat, off, w, [1, 2, 5, 10, 50, 100, 10 ** 6])
    assert np.all(np.diff(out) >= 0)
    assert out[-1] == 1.0 and out[-2] == 1.0


def test_weight_scale_invariance(oracle):
    sc, lat, off, w = inputs.make_eval_tasks(20, 6, max_len=200)
    a, _, _ = oracle.topk_score(sc, lat, off, w, [1, 5])
    b, _, _ = oracle.topk_score(sc, lat, off, w * 4, [1, 5])
    np.testing.assert_allclose(a, b, rtol=1e-15)


def _brute(sc, lat, off, w, k):
    num = den = 0.0
    for t in range(len(off) - 1):
        s = sc[off[t]:off[t + 1]].astype(np.float64)
        s = np.where(np.isnan(s), -np.inf, s)
        l = lat[off[t]:off[t + 1]].astype(np.float64)
        order = np.lexsort((np.arange(s.size), -s))     # score desc, index asc
        num += l.min() * w[t]
        den += l[order[:k]].min() * w[t]
    return num / den


@pytest.mark.parametrize("seed,tq", [(0, 0.0), (1, 0.25), (2, 1.0)])
def test_brute_force(oracle, seed, tq):
    sc, lat, off, w = inputs.make_eval_tasks(100, seed, max_len=400, tie_quant=tq)
    sc[::37] = np.nan
    ks = [1, 3, 5, 10]
    out, _, _ = oracle.topk_score(sc, lat, off, w, ks)
    for j, k in enumerate(ks):
        assert out[j] == pytest.approx(_brute(sc, lat, off, w, k), rel=1e-12)
