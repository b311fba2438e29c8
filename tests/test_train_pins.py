"""Pins of the training-step oracle (oracle/train_oracle.py; Eq. 6, §7.1.3; reading R24).

* its fp64 torch forward equals the (separately pinned) C oracle to 1e-12;
* LambdaRank: SPEC's worked cases (equal scores -> the pair term is dNDCG; the inverted two-item
  group evaluated by hand), invariance to a common shift and to member order, the large-margin
  limit;
* parameter gradients (autograd) against central finite differences of the C oracle's scores
  pushed through the loss;
* the Adam step against its closed form at t = 1 (|update| = lr for every nonzero gradient).
"""
import math

import numpy as np
import pytest

import inputs
from oracle import train_oracle as TO


def _tiny(n=6, seed=3):
    c = inputs.config("tiny")
    d = c["dims"]
    w = inputs.make_weights(d, c["seed"])
    f, l = inputs.make_features(d, n, seed)
    return d, w, f, l


def test_torch_forward_matches_c_oracle(oracle):
    for name in ("tiny", "tuning"):
        c = inputs.config(name)
        d = c["dims"]
        w = inputs.make_weights(d, c["seed"])
        f, l = inputs.make_features(d, 5, 11)
        s = TO.forward(d, TO.params_from_blob(d, w), f, l).detach().numpy()
        np.testing.assert_allclose(s, oracle.score(d, w, f, l), rtol=1e-12, atol=1e-12)


def test_equal_scores_pair_is_dndcg():
    # SPEC: s_i == s_j -> pair term = dNDCG * log2(2) = dNDCG.  Two items, y = [1, 0.5]:
    # ranks by (score desc, index asc) -> item 0 rank 1, item 1 rank 2.
    loss, _ = TO.loss_and_score_grad(np.array([0.3, 0.3]), np.float32([1.0, 2.0]), np.array([0, 2]))
    g = np.array([1.0, math.sqrt(2.0) - 1.0])            # 2^y - 1
    max_dcg = g[0] / math.log2(2) + g[1] / math.log2(3)  # ideal order = item 0 first
    dndcg = abs(g[0] - g[1]) / max_dcg * abs(1 / math.log2(2) - 1 / math.log2(3))
    assert loss == pytest.approx(dndcg, rel=1e-14)


def test_inverted_two_item_group_by_hand():
    # SPEC: y = [1.0, 0.5], scores [1.0, 2.0] (inverted): item 1 ranked first.
    loss, grad = TO.loss_and_score_grad(np.array([1.0, 2.0]), np.float32([1.0, 2.0]), np.array([0, 2]))
    g = np.array([1.0, math.sqrt(2.0) - 1.0])
    max_dcg = g[0] + g[1] / math.log2(3)
    D = np.array([math.log2(3), 1.0])                    # item 0 at rank 2, item 1 at rank 1
    dndcg = abs(g[0] - g[1]) / max_dcg * abs(1 / D[0] - 1 / D[1])
    assert loss == pytest.approx(dndcg * math.log2(1 + math.exp(1.0)), rel=1e-14)
    # LambdaRank gradient: dL/ds_0 = -dndcg * sigmoid(-(s_0 - s_1)) / ln 2 = -dL/ds_1
    lam = dndcg / (1 + math.exp(-1.0)) / math.log(2)
    np.testing.assert_allclose(grad, [-lam, lam], rtol=1e-13)


def test_loss_invariances():
    rng = np.random.default_rng(0)
    sc = rng.normal(size=40)
    lat = np.exp(rng.normal(size=40)).astype(np.float32)
    off = np.array([0, 13, 40])
    base, _ = TO.loss_and_score_grad(sc, lat, off)
    shifted, _ = TO.loss_and_score_grad(sc + np.r_[np.full(13, 5.0), np.full(27, -2.0)], lat, off)
    assert shifted == pytest.approx(base, rel=1e-12)
    perm = np.r_[rng.permutation(13), 13 + rng.permutation(27)]
    permuted, _ = TO.loss_and_score_grad(sc[perm], lat[perm], off)
    assert permuted == pytest.approx(base, rel=1e-12)
    # perfectly ordered (score = -log latency) with a large margin -> loss -> 0
    far, _ = TO.loss_and_score_grad(-5000.0 * np.log(lat.astype(np.float64)), lat, off)
    assert far < 1e-6 * base


def test_gradients_against_finite_differences(oracle):
    d, w, f, l = _tiny(n=6)
    lat = np.exp(np.random.default_rng(1).normal(size=6)).astype(np.float32)
    off = np.array([0, 4, 6])
    loss, grad, _, _ = TO.train_grads(d, w, f, l, lat, off)

    def loss_of(wb):   # C-oracle scores (independent forward) through the loss
        return TO.loss_and_score_grad(oracle.score(d, wb.astype(np.float32), f, l), lat, off)[0]

    rng = np.random.default_rng(2)
    man = inputs.manifest(d)
    checked = 0
    for m in man:       # a few coordinates of every tensor
        cnt = int(np.prod(m["shape"]))
        for k in rng.choice(cnt, size=min(2, cnt), replace=False):
            i = m["offset"] + int(k)
            h = 1e-3 * max(1.0, abs(float(w[i])))
            wp, wm = w.astype(np.float64).copy(), w.astype(np.float64).copy()
            wp[i] += h
            wm[i] -= h
            # fp32 weights: use a step exactly representable around w[i]
            wp32, wm32 = wp.astype(np.float32), wm.astype(np.float32)
            hh = (float(wp32[i]) - float(wm32[i])) / 2
            fd = (loss_of(wp32) - loss_of(wm32)) / (2 * hh)
            assert abs(fd - grad[i]) <= 2e-4 * max(1e-3, abs(grad[i])) + 1e-7, (m["name"], k, fd, grad[i])
            checked += 1
    assert checked >= len(man)


def test_adam_first_step_closed_form():
    rng = np.random.default_rng(4)
    w = rng.normal(size=50)
    g = rng.normal(size=50)
    g[::7] = 0.0
    w1, m1, v1 = TO.adam_step(w, g, np.zeros(50), np.zeros(50), 1, lr=7e-4, eps=1e-300)
    step = w - w1
    np.testing.assert_allclose(np.abs(step[g != 0]), 7e-4, rtol=1e-12)
    assert np.all(np.sign(step[g != 0]) == np.sign(g[g != 0]))
    assert np.all(step[g == 0] == 0)
