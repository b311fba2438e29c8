"""ctypes binding of the fp64 CPU oracle (oracle/tcl_oracle.c).

TEST INFRASTRUCTURE ONLY: only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / `--impl reference` legs may import this module.  The product path
(paper_2604_12891_b200/) never imports it; the two share no code.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from typing import Dict, Optional, Tuple

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "tcl_oracle.c")
LIB = os.path.join(HERE, "libtcl_oracle.so")


def build(force: bool = False) -> str:
    """gcc -O2, no -march, no BLAS, no intrinsics: the 'plain, slow' baseline."""
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        tmp = LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-ffp-contract=off", "-Wall", "-shared", "-fPIC", "-pthread",
                               "-o", tmp, SRC, "-lm"])
        os.replace(tmp, LIB)
    return LIB


class _Dims(ctypes.Structure):
    _fields_ = [("d_in", ctypes.c_int32), ("max_len", ctypes.c_int32), ("d_model", ctypes.c_int32),
                ("n_layer", ctypes.c_int32), ("d_state", ctypes.c_int32), ("d_conv", ctypes.c_int32),
                ("expand", ctypes.c_int32), ("dt_rank", ctypes.c_int32),
                ("enc_dims", ctypes.c_int32 * 3), ("dec_dims", ctypes.c_int32 * 3),
                ("ln_eps", ctypes.c_float), ("dropout_p", ctypes.c_float),
                ("precision", ctypes.c_int32), ("disc", ctypes.c_int32)]


def _cdims(d) -> _Dims:
    return _Dims(d.d_in, d.max_len, d.d_model, d.n_layer, d.d_state, d.d_conv, d.expand, d.dt_rank,
                 (ctypes.c_int32 * 3)(*d.enc_dims), (ctypes.c_int32 * 3)(*d.dec_dims),
                 d.ln_eps, d.dropout_p, d.precision, d.disc)


_lib: Optional[ctypes.CDLL] = None


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        L = ctypes.CDLL(build())
        P = ctypes.POINTER
        dp = P(ctypes.c_double)
        fp = P(ctypes.c_float)
        ip = P(ctypes.c_int32)
        lp = P(ctypes.c_int64)
        L.tclo_silu.restype = ctypes.c_double
        L.tclo_silu.argtypes = [ctypes.c_double]
        L.tclo_softplus.restype = ctypes.c_double
        L.tclo_softplus.argtypes = [ctypes.c_double]
        L.tclo_weights_count.restype = ctypes.c_int64
        L.tclo_weights_count.argtypes = [P(_Dims)]
        L.tclo_dump_size.restype = ctypes.c_int64
        L.tclo_dump_size.argtypes = [P(_Dims), ctypes.c_int]
        L.tclo_layernorm_row.argtypes = [dp, ctypes.c_int, fp, fp, ctypes.c_double, dp]
        L.tclo_causal_conv_silu.argtypes = [dp, ctypes.c_int, ctypes.c_int, ctypes.c_int, fp, fp, dp]
        L.tclo_ssm_scan.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, dp, dp, dp, dp, dp, dp,
                                    ctypes.c_int, dp]
        L.tclo_philox4x32_10.argtypes = [P(ctypes.c_uint32), P(ctypes.c_uint32), P(ctypes.c_uint32)]
        L.tclo_forward_one.argtypes = [P(_Dims), fp, fp, ctypes.c_int, dp, dp]
        L.tclo_score.argtypes = [P(_Dims), fp, fp, ip, ctypes.c_int64, dp, ctypes.c_int]
        L.tclo_score_mc.argtypes = [P(_Dims), fp, fp, ip, ctypes.c_int64, ctypes.c_int32,
                                    ctypes.c_uint64, ctypes.c_int64, dp, dp, ctypes.c_int]
        L.tclo_score_pass.argtypes = [P(_Dims), fp, fp, ip, ctypes.c_int64, ctypes.c_int32, ctypes.c_uint64,
                                      ctypes.c_int64, dp, ctypes.c_int]
        L.tclo_topk_f64.argtypes = [dp, ctypes.c_int64, ctypes.c_int32, ctypes.c_int64, lp, dp]
        L.tclo_topk_f32.argtypes = [fp, ctypes.c_int64, ctypes.c_int32, ctypes.c_int64, lp, fp]
        L.tclo_adapters_count.restype = ctypes.c_int64
        L.tclo_adapters_count.argtypes = [P(_Dims), ctypes.c_int]
        L.tclo_score_kbac.argtypes = [P(_Dims), fp, fp, fp, ctypes.c_int, fp, ip, ctypes.c_int64, dp, ctypes.c_int]
        L.tclo_score_mc_kbac.argtypes = [P(_Dims), fp, fp, fp, ctypes.c_int, fp, ip, ctypes.c_int64, ctypes.c_int32,
                                         ctypes.c_uint64, ctypes.c_int64, dp, dp, ctypes.c_int]
        L.tclo_topk_score.argtypes = [fp, fp, lp, fp, ctypes.c_int64, ip, ctypes.c_int32, dp, dp, dp]
        L.tclo_rdu_scores.argtypes = [fp, ctypes.c_int64, fp, ctypes.c_int64, fp, fp, fp]
        L.tclo_rdu_select.restype = ctypes.c_int64
        L.tclo_rdu_select.argtypes = [fp, ip, ctypes.c_int64, fp, ctypes.c_int64, ctypes.c_int32, ctypes.c_int32, lp]
        _lib = L
    return _lib


def _p(a: np.ndarray, ct):
    return a.ctypes.data_as(ctypes.POINTER(ct))


def _f32(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float32)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def silu(v: float) -> float:
    return lib().tclo_silu(float(v))


def softplus(v: float) -> float:
    return lib().tclo_softplus(float(v))


def weights_count(d) -> int:
    return int(lib().tclo_weights_count(ctypes.byref(_cdims(d))))


def layernorm(x: np.ndarray, g: Optional[np.ndarray] = None, b: Optional[np.ndarray] = None,
              eps: float = 1e-5) -> np.ndarray:
    x = _f64(np.atleast_2d(x))
    y = np.empty_like(x)
    gg = _f32(g) if g is not None else None
    bb = _f32(b) if b is not None else None
    for r in range(x.shape[0]):
        lib().tclo_layernorm_row(_p(x[r], ctypes.c_double), x.shape[1],
                                 _p(gg, ctypes.c_float) if gg is not None else None,
                                 _p(bb, ctypes.c_float) if bb is not None else None, eps,
                                 _p(y[r], ctypes.c_double))
    return y


def causal_conv_silu(x: np.ndarray, w: np.ndarray, b: Optional[np.ndarray]) -> np.ndarray:
    x = _f64(x)
    T, di = x.shape
    w = _f32(w)
    c = np.empty_like(x)
    bb = _f32(b) if b is not None else None
    lib().tclo_causal_conv_silu(_p(x, ctypes.c_double), T, di, w.shape[1], _p(w, ctypes.c_float),
                                _p(bb, ctypes.c_float) if bb is not None else None,
                                _p(c, ctypes.c_double))
    return c


def ssm_scan(u, delta, A, B, C, Dv, disc: int = 0) -> np.ndarray:
    u, delta, A, B, C, Dv = map(_f64, (u, delta, A, B, C, Dv))
    T, di = u.shape
    N = A.shape[1]
    y = np.empty_like(u)
    lib().tclo_ssm_scan(T, di, N, *[_p(a, ctypes.c_double) for a in (u, delta, A, B, C, Dv)], disc,
                        _p(y, ctypes.c_double))
    return y


def philox4x32_10(ctr, key) -> np.ndarray:
    c = np.ascontiguousarray(ctr, dtype=np.uint32)
    k = np.ascontiguousarray(key, dtype=np.uint32)
    o = np.zeros(4, dtype=np.uint32)
    lib().tclo_philox4x32_10(_p(c, ctypes.c_uint32), _p(k, ctypes.c_uint32), _p(o, ctypes.c_uint32))
    return o


def forward_one(d, w: np.ndarray, feats_one: np.ndarray, T: int) -> Tuple[float, Dict[str, np.ndarray]]:
    """Score of one candidate plus every intermediate (per-stage dumps)."""
    cd = _cdims(d)
    w = _f32(w)
    x = _f32(feats_one)
    size = int(lib().tclo_dump_size(ctypes.byref(cd), T))
    dump = np.zeros(size, dtype=np.float64)
    s = ctypes.c_double(0)
    rc = lib().tclo_forward_one(ctypes.byref(cd), _p(w, ctypes.c_float), _p(x, ctypes.c_float), T,
                                _p(dump, ctypes.c_double), ctypes.byref(s))
    if rc != 0:
        raise ValueError("tclo_forward_one failed")
    dm, di, N, R = d.d_model, d.d_inner, d.d_state, d.dt_rank
    out, off = {}, 0

    def take(name, shape):
        nonlocal off
        cnt = int(np.prod(shape))
        out[name] = dump[off:off + cnt].reshape(shape)
        off += cnt

    take("h_enc", (T, dm))
    for l in range(d.n_layer):
        for nm, shp in (("a", (T, dm)), ("x", (T, di)), ("z", (T, di)), ("u", (T, di)),
                        ("dtr", (T, R)), ("B", (T, N)), ("C", (T, N)), ("delta", (T, di)),
                        ("y", (T, di)), ("g", (T, di)), ("h", (T, dm))):
            take(f"layer{l}.{nm}", shp)
    take("pooled", (dm,))
    take("dec_h1", (d.dec_dims[0],))
    take("dec_h2", (d.dec_dims[1],))
    assert off == size
    return float(s.value), out


def default_threads() -> int:
    return max(1, os.cpu_count() or 1)


def score(d, w: np.ndarray, feats: np.ndarray, lens: np.ndarray, nthreads: Optional[int] = None) -> np.ndarray:
    feats = _f32(feats)
    lens = np.ascontiguousarray(lens, dtype=np.int32)
    n = lens.shape[0]
    assert feats.shape == (n, d.max_len, d.d_in), feats.shape
    out = np.zeros(n, dtype=np.float64)
    rc = lib().tclo_score(ctypes.byref(_cdims(d)), _p(_f32(w), ctypes.c_float), _p(feats, ctypes.c_float),
                          _p(lens, ctypes.c_int32), n, _p(out, ctypes.c_double),
                          nthreads or default_threads())
    if rc != 0:
        raise ValueError("tclo_score failed")
    return out


def score_mc(d, w, feats, lens, n_passes: int, seed: int, index_base: int = 0,
             nthreads: Optional[int] = None) -> Tuple[np.ndarray, np.ndarray]:
    feats = _f32(feats)
    lens = np.ascontiguousarray(lens, dtype=np.int32)
    n = lens.shape[0]
    mean = np.zeros(n, dtype=np.float64)
    var = np.zeros(n, dtype=np.float64)
    rc = lib().tclo_score_mc(ctypes.byref(_cdims(d)), _p(_f32(w), ctypes.c_float), _p(feats, ctypes.c_float),
                             _p(lens, ctypes.c_int32), n, n_passes, seed, index_base,
                             _p(mean, ctypes.c_double), _p(var, ctypes.c_double), nthreads or default_threads())
    if rc != 0:
        raise ValueError("tclo_score_mc failed")
    return mean, var


def score_pass(d, w, feats, lens, pass_index: int, seed: int, index_base: int = 0,
               nthreads: Optional[int] = None) -> np.ndarray:
    """Scores of ONE MC-dropout pass (the masks tclo_score_mc uses for that pass)."""
    feats = _f32(feats)
    lens = np.ascontiguousarray(lens, dtype=np.int32)
    n = lens.shape[0]
    out = np.zeros(n, dtype=np.float64)
    rc = lib().tclo_score_pass(ctypes.byref(_cdims(d)), _p(_f32(w), ctypes.c_float), _p(feats, ctypes.c_float),
                               _p(lens, ctypes.c_int32), n, pass_index, seed, index_base,
                               _p(out, ctypes.c_double), nthreads or default_threads())
    if rc != 0:
        raise ValueError("tclo_score_pass failed")
    return out


def topk(scores: np.ndarray, k: int, index_base: int = 0) -> Tuple[np.ndarray, np.ndarray]:
    """(idx int64 [k], score [k]) under (score desc, index asc), NaN -> -inf, clamp + fill."""
    idx = np.zeros(k, dtype=np.int64)
    if scores.dtype == np.float32:
        s = _f32(scores)
        top = np.zeros(k, dtype=np.float32)
        rc = lib().tclo_topk_f32(_p(s, ctypes.c_float), s.shape[0], k, index_base,
                                 _p(idx, ctypes.c_int64), _p(top, ctypes.c_float))
    else:
        s = _f64(scores)
        top = np.zeros(k, dtype=np.float64)
        rc = lib().tclo_topk_f64(_p(s, ctypes.c_double), s.shape[0], k, index_base,
                                 _p(idx, ctypes.c_int64), _p(top, ctypes.c_double))
    if rc != 0:
        raise ValueError("topk failed")
    return idx, top


def rdu_select(pool_scores, pool_ops, labeled_scores, n_ops: int, budget_total: int) -> np.ndarray:
    """One RDU selection round (Alg. 1 lines 16-31, Eqs. 1-3): indices of the picks, in order."""
    ps = _f32(pool_scores)
    po = np.ascontiguousarray(pool_ops, dtype=np.int32)
    ls = _f32(labeled_scores) if len(labeled_scores) else np.zeros(1, np.float32)
    out = np.zeros(max(1, budget_total), dtype=np.int64)
    k = lib().tclo_rdu_select(_p(ps, ctypes.c_float), _p(po, ctypes.c_int32), ps.shape[0],
                              _p(ls, ctypes.c_float), len(labeled_scores), n_ops, budget_total,
                              _p(out, ctypes.c_int64))
    return out[:k]


def _rdu_prepare_f64(pool_scores, pool_ops, labeled_scores, n_ops: int, budget_total: int):
    """Alg. 1 lines 16-19 in fp64: f^ (min-max over finite pool u labeled predictions, 0.5 when
    flat), eligibility (finite, op in range) and the per-op budgets B_t count(op) / n_pool."""
    pool = np.asarray(pool_scores, dtype=np.float64)
    ops = np.asarray(pool_ops, dtype=np.int64)
    lab = np.asarray(labeled_scores, dtype=np.float64)
    fin = np.concatenate([pool[np.isfinite(pool)], lab[np.isfinite(lab)]])
    lo, hi = (fin.min(), fin.max()) if fin.size else (0.0, 0.0)
    norm = (lambda v: np.full_like(v, 0.5)) if not hi > lo else (lambda v: (v - lo) / (hi - lo))
    fh = norm(pool)
    labh = list(norm(lab[np.isfinite(lab)]))
    ok_op = (ops >= 0) & (ops < n_ops)
    alive = np.isfinite(pool) & ok_op
    count = np.bincount(ops[ok_op], minlength=n_ops).astype(np.float64)
    budget = budget_total * count / pool.size
    return fh, ops, labh, alive, budget


def _rdu_total_f64(fh, labh):
    """Eq. 1 (d_s: nearest labeled f^, 1 when none), Eqs. 2-3 (u_s: population variance of the
    labeled set plus the candidate, TWO-PASS: mean first, then the squared deviations) and line 24
    (t_s = f^ d_s + u_s), all in fp64, for every candidate f^ in `fh`."""
    L = np.asarray(labh, dtype=np.float64)
    if L.size == 0:
        return fh * 1.0 + 0.0
    ds = np.abs(fh[:, None] - L[None, :]).min(1)
    mu = (fh + L.sum()) / (L.size + 1)
    us = ((fh - mu) ** 2 + ((L[None, :] - mu[:, None]) ** 2).sum(1)) / (L.size + 1)
    return fh * ds + us


def rdu_select_f64(pool_scores, pool_ops, labeled_scores, n_ops: int, budget_total: int) -> np.ndarray:
    """One RDU selection round (Alg. 1 lines 16-31, Eqs. 1-3) written plainly in fp64: every pick
    recomputes d_s and the two-pass variance over the current labeled set; argmax t_s, ties by
    higher f^ then lower index (reading R21); a pick joins the labeled set before the next."""
    fh, ops, labh, alive, budget = _rdu_prepare_f64(pool_scores, pool_ops, labeled_scores, n_ops, budget_total)
    sel = np.zeros(n_ops)
    picks = []
    for _ in range(budget_total):
        elig = alive.copy()
        elig[alive] = sel[ops[alive]] < budget[ops[alive]]
        idx = np.nonzero(elig)[0]
        if idx.size == 0:
            break
        t = _rdu_total_f64(fh[idx], labh)
        best = idx[np.lexsort((idx, -fh[idx], -t))[0]]
        picks.append(int(best))
        alive[best] = False
        sel[ops[best]] += 1
        labh.append(fh[best])
    return np.array(picks, dtype=np.int64)


def rdu_follow_f64(pool_scores, pool_ops, labeled_scores, n_ops: int, budget_total: int, picks,
                   tol: float) -> int:
    """Replay a pick sequence (e.g. the GPU's) in fp64 (R19-style near-tie rule for RDU): every pick
    must be eligible and its fp64 t_s within `tol` of the best eligible fp64 t_s given the picks
    before it; the sequence may only end when nothing is eligible.  Returns the number of picks
    that are not the fp64 argmax (near ties, each within tol); raises AssertionError otherwise."""
    fh, ops, labh, alive, budget = _rdu_prepare_f64(pool_scores, pool_ops, labeled_scores, n_ops, budget_total)
    sel = np.zeros(n_ops)
    near = 0
    for step in range(budget_total):
        elig = alive.copy()
        elig[alive] = sel[ops[alive]] < budget[ops[alive]]
        idx = np.nonzero(elig)[0]
        if step == len(picks):
            assert idx.size == 0, f"sequence ended after {step} picks with {idx.size} eligible candidates"
            break
        if idx.size == 0:
            raise AssertionError(f"pick {step} made with no eligible candidate")
        b = int(picks[step])
        assert elig[b], f"pick {step} ({b}) is not eligible"
        t = _rdu_total_f64(fh[idx], labh)
        best = idx[np.lexsort((idx, -fh[idx], -t))[0]]
        tb = t[np.searchsorted(idx, b)]
        assert tb >= t.max() - tol, f"pick {step}: t_s {tb:.9g} < best {t.max():.9g} - {tol}"
        near += int(b != best)
        alive[b] = False
        sel[ops[b]] += 1
        labh.append(fh[b])
    return near


def rdu_scores(fh_pool, fh_lab):
    """(d_s, u_s, t_s) of Eqs. 1-3 / line 24 for already-normalised predictions (fp32)."""
    fp_ = _f32(fh_pool)
    fl = _f32(fh_lab) if len(fh_lab) else np.zeros(1, np.float32)
    ds, us, ts = (np.zeros(fp_.shape[0], np.float32) for _ in range(3))
    lib().tclo_rdu_scores(_p(fp_, ctypes.c_float), fp_.shape[0], _p(fl, ctypes.c_float), len(fh_lab),
                          _p(ds, ctypes.c_float), _p(us, ctypes.c_float), _p(ts, ctypes.c_float))
    return ds, us, ts


def topk_score(scores, latency, task_offsets, task_weights, ks):
    """Eq. 12 Top-k score for each k in ks: (score[], num[], den[]) in fp64."""
    sc, la = _f32(scores), _f32(latency)
    off = np.ascontiguousarray(task_offsets, dtype=np.int64)
    w = _f32(task_weights)
    kk = np.ascontiguousarray(ks, dtype=np.int32)
    out, num, den = (np.zeros(kk.size) for _ in range(3))
    rc = lib().tclo_topk_score(_p(sc, ctypes.c_float), _p(la, ctypes.c_float), _p(off, ctypes.c_int64),
                               _p(w, ctypes.c_float), off.size - 1, _p(kk, ctypes.c_int32), kk.size,
                               _p(out, ctypes.c_double), _p(num, ctypes.c_double), _p(den, ctypes.c_double))
    if rc != 0:
        raise ValueError("tclo_topk_score: bad arguments")
    return out, num, den


def adapters_count(d, a: int) -> int:
    """Floats in the KB+AC adapter blob of rank a (Eq. 7 sites, reading R23)."""
    return int(lib().tclo_adapters_count(ctypes.byref(_cdims(d)), a))


def score_kbac(d, kb_w, ac_w, ad_w, a: int, feats, lens, nthreads: Optional[int] = None) -> np.ndarray:
    """KB + AC two-column scores (Eq. 7 lateral adapters; the AC column's output)."""
    feats = _f32(feats)
    lens = np.ascontiguousarray(lens, dtype=np.int32)
    n = lens.shape[0]
    out = np.zeros(n, dtype=np.float64)
    rc = lib().tclo_score_kbac(ctypes.byref(_cdims(d)), _p(_f32(kb_w), ctypes.c_float), _p(_f32(ac_w), ctypes.c_float),
                               _p(_f32(ad_w), ctypes.c_float), a, _p(feats, ctypes.c_float),
                               _p(lens, ctypes.c_int32), n, _p(out, ctypes.c_double), nthreads or default_threads())
    if rc != 0:
        raise ValueError("tclo_score_kbac failed")
    return out


def score_mc_kbac(d, kb_w, ac_w, ad_w, a: int, feats, lens, n_passes: int, seed: int, index_base: int = 0,
                  nthreads: Optional[int] = None) -> Tuple[np.ndarray, np.ndarray]:
    feats = _f32(feats)
    lens = np.ascontiguousarray(lens, dtype=np.int32)
    n = lens.shape[0]
    mean = np.zeros(n, dtype=np.float64)
    var = np.zeros(n, dtype=np.float64)
    rc = lib().tclo_score_mc_kbac(ctypes.byref(_cdims(d)), _p(_f32(kb_w), ctypes.c_float),
                                  _p(_f32(ac_w), ctypes.c_float), _p(_f32(ad_w), ctypes.c_float), a,
                                  _p(feats, ctypes.c_float), _p(lens, ctypes.c_int32), n, n_passes, seed,
                                  index_base, _p(mean, ctypes.c_double), _p(var, ctypes.c_double),
                                  nthreads or default_threads())
    if rc != 0:
        raise ValueError("tclo_score_mc_kbac failed")
    return mean, var
