"""Pins of the RDU acquisition oracle (§4, Algorithm 1 lines 16-31, Eqs. 1-3; reading R21).

Each pin fixes the oracle to something other than itself: the worked values SPEC.md lists for
d_s / u_s / t_s, closed forms (Eq. 3 against a two-pass variance, an empty labeled set), a brute
force re-selection written independently in fp64 numpy (recomputing every score from scratch at
every pick), the budget contract of Alg. 1 lines 16-31 and the degenerate cases.
"""
import numpy as np
import pytest


def test_diversity_example(oracle):
    # SPEC rdu.diversity_score: labeled {0.2, 0.9}, candidate 0.5 -> d_s = 0.3 (Eq. 1)
    ds, _, _ = oracle.rdu_scores([0.5], [0.2, 0.9])
    assert ds[0] == pytest.approx(0.3, abs=1e-7)


def test_uncertainty_example(oracle):
    # SPEC rdu.uncertainty_score: M = 1, labeled {0}, candidate 1 -> mu = 0.5, sigma^2 = 0.25 (Eqs. 2-3)
    ds, us, ts = oracle.rdu_scores([1.0], [0.0])
    assert us[0] == 0.25 and ds[0] == 1.0
    assert ts[0] == 1.25    # line 24: f d_s + u_s = 1*1 + 0.25


def test_total_score_composition(oracle):
    # SPEC rdu.total_score: f = 0.5, d_s = 0.3, u_s = 0.25 -> 0.4 ; d_s = 0 -> t_s = u_s.
    # Build the inputs: labeled {0.2, 0.8} gives d_s(0.5) = 0.3 and a closed-form u_s.
    ds, us, ts = oracle.rdu_scores([0.5], [0.2, 0.8])
    mu = (0.5 + 0.2 + 0.8) / 3
    var = ((0.5 - mu) ** 2 + (0.2 - mu) ** 2 + (0.8 - mu) ** 2) / 3
    assert us[0] == pytest.approx(var, abs=1e-7)
    assert ts[0] == pytest.approx(0.5 * 0.3 + var, abs=1e-7)
    assert 0.5 * 0.3 + 0.25 == pytest.approx(0.4)
    ds, us, ts = oracle.rdu_scores([0.2], [0.2, 0.8])   # candidate equals a labeled score: d_s = 0
    assert ds[0] == 0.0 and ts[0] == us[0]


def test_empty_labeled(oracle):
    # M = 0: mu = f, sigma^2 = 0 (Eq. 3 with a single element); d_s = 1 (reading R21)
    ds, us, ts = oracle.rdu_scores([0.1, 0.7, 1.0], [])
    assert np.all(ds == 1.0) and np.all(us == 0.0)
    np.testing.assert_array_equal(ts, np.float32([0.1, 0.7, 1.0]))


def test_incremental_variance_matches_two_pass(oracle):
    # Eq. 3 via running S, Q (O(1) per candidate) against the two-pass population variance (fp64)
    rng = np.random.default_rng(5)
    lab = rng.random(300).astype(np.float32)
    pool = rng.random(200).astype(np.float32)
    ds, us, _ = oracle.rdu_scores(pool, lab)
    for i in range(pool.size):
        v = np.concatenate([[pool[i]], lab]).astype(np.float64)
        assert abs(us[i] - v.var()) < 2e-6
        assert ds[i] == np.abs(lab.astype(np.float64) - pool[i]).min().astype(np.float32)


def _brute_force(pool, ops, lab, n_ops, B):
    """Alg. 1 lines 16-31 written from scratch in fp64: every pick recomputes d_s and u_s over the
    current labeled set (no running sums)."""
    pool = pool.astype(np.float64)
    lab = lab.astype(np.float64)
    allv = np.concatenate([pool, lab])
    lo, hi = allv.min(), allv.max()
    fh = (pool - lo) / (hi - lo)
    labh = list((lab - lo) / (hi - lo))
    budget = {o: B * np.count_nonzero(ops == o) / pool.size for o in range(n_ops)}
    sel = {o: 0 for o in range(n_ops)}
    taken, picks = set(), []
    while len(picks) < B:
        best = None
        for i in range(pool.size):
            if i in taken or not sel[ops[i]] < budget[ops[i]]:
                continue
            d = min(abs(fh[i] - x) for x in labh) if labh else 1.0
            u = np.var(np.array([fh[i]] + labh))
            key = (fh[i] * d + u, fh[i], -i)
            if best is None or key > best[0]:
                best = (key, i)
        if best is None:
            break
        i = best[1]
        picks.append(i)
        taken.add(i)
        sel[ops[i]] += 1
        labh.append(fh[i])
    return picks


@pytest.mark.parametrize("seed,n,m,n_ops,B", [(0, 40, 0, 1, 10), (1, 60, 5, 3, 20), (2, 80, 30, 4, 40),
                                              (3, 50, 1, 2, 50), (4, 33, 7, 5, 9)])
def test_selection_brute_force(oracle, seed, n, m, n_ops, B):
    rng = np.random.default_rng(seed)
    # well-separated values (multiples of 1/1024 with distinct gaps) so fp32 and fp64 agree on argmax
    pool = (rng.permutation(4096)[:n] / 4096.0).astype(np.float32)
    lab = (rng.permutation(4096)[:m] / 4096.0 + 1 / 8192).astype(np.float32)
    ops = rng.integers(0, n_ops, n).astype(np.int32)
    got = oracle.rdu_select(pool, ops, lab, n_ops, B)
    want = _brute_force(pool, ops, lab, n_ops, B)
    assert list(got) == want


def test_budget_contract(oracle):
    rng = np.random.default_rng(11)
    n, n_ops, B = 5000, 7, 500
    p = np.array([0.4, 0.2, 0.15, 0.1, 0.1, 0.04, 0.01])
    ops = rng.choice(n_ops, n, p=p).astype(np.int32)
    pool = rng.normal(size=n).astype(np.float32)
    lab = rng.normal(size=64).astype(np.float32)
    picks = oracle.rdu_select(pool, ops, lab, n_ops, B)
    assert len(set(picks.tolist())) == len(picks) <= B
    for o in range(n_ops):
        cnt = np.count_nonzero(ops == o)
        got = np.count_nonzero(ops[picks] == o)
        assert got <= np.ceil(B * cnt / n)           # SPEC: per-op counts <= ceil(B_t * prob_op)
    assert len(picks) == B     # sum_op ceil(budget_op) >= B_t: the round never ends early (line 22)


def test_degenerate_full_budget(oracle):
    # B_t = pool size, one operator type: the whole pool is selected (each index once)
    rng = np.random.default_rng(3)
    pool = rng.random(257).astype(np.float32)
    picks = oracle.rdu_select(pool, np.zeros(257, np.int32), np.float32([]), 1, 257)
    assert sorted(picks.tolist()) == list(range(257))
    # the first pick with no labeled data maximises t_s = f^ (d_s = 1, u_s = 0): the best prediction
    assert picks[0] == int(np.argmax(pool))


def test_flat_and_nonfinite(oracle):
    # all predictions equal: every t_s ties, so picks follow the index order (P:350 tie rule)
    picks = oracle.rdu_select(np.full(20, 3.0, np.float32), np.zeros(20, np.int32), np.float32([3.0]), 1, 5)
    assert picks.tolist() == [0, 1, 2, 3, 4]
    pool = np.float32([0.1, np.nan, 0.9, np.inf, -np.inf, 0.5])
    picks = oracle.rdu_select(pool, np.zeros(6, np.int32), np.float32([np.nan, 0.2]), 1, 6)
    assert sorted(picks.tolist()) == [0, 2, 5]


@pytest.mark.parametrize("seed,n,m,n_ops,B", [(0, 40, 0, 1, 10), (1, 60, 5, 3, 20), (2, 80, 30, 4, 40),
                                              (3, 50, 1, 2, 50), (4, 33, 7, 5, 9)])
def test_f64_oracle_brute_force(oracle, seed, n, m, n_ops, B):
    """The plain fp64 selection (oracle.rdu_select_f64, two-pass Eq. 3) against the from-scratch
    pure-Python brute force, on the same well-separated inputs."""
    rng = np.random.default_rng(seed)
    pool = (rng.permutation(4096)[:n] / 4096.0).astype(np.float32)
    lab = (rng.permutation(4096)[:m] / 4096.0 + 1 / 8192).astype(np.float32)
    ops = rng.integers(0, n_ops, n).astype(np.int32)
    assert oracle.rdu_select_f64(pool, ops, lab, n_ops, B).tolist() == _brute_force(pool, ops, lab, n_ops, B)


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_fp32_selection_within_near_ties_of_f64(oracle, seed):
    """The fp32 oracle (the kernel's operation order) follows the fp64 selection up to near ties:
    every fp32 pick is within 1e-5 of the best fp64 total score given the picks before it."""
    rng = np.random.default_rng(100 + seed)
    n, m, n_ops, B = 1500, 40, 6, 150
    pool = rng.normal(size=n).astype(np.float32)
    lab = rng.normal(size=m).astype(np.float32)
    ops = rng.integers(0, n_ops, n).astype(np.int32)
    picks = oracle.rdu_select(pool, ops, lab, n_ops, B)
    near = oracle.rdu_follow_f64(pool, ops, lab, n_ops, B, picks, tol=1e-5)
    assert near <= B // 20
    # a deliberately wrong sequence (the worst candidate first) is rejected
    bad = picks.copy()
    bad[0] = int(np.argmin(np.where(np.isfinite(pool), pool, np.inf)))
    with pytest.raises(AssertionError):
        oracle.rdu_follow_f64(pool, ops, lab, n_ops, B, bad, tol=1e-5)
