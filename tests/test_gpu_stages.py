"""Per-stage GPU parity (SURVEY §4 tier T2): the workspace buffers of a 1-layer model, read back
through tcl_debug_read, against the oracle's per-stage dumps of the same candidates.

bf16 path: operands are rounded to bf16 (8-bit mantissa), so stage tolerances are relative to the
stage's magnitude: |gpu - ref| <= rtol * max|ref| + rtol * |ref| with rtol = 2e-2 (the north-star
bf16 bound); the fp32 path is checked at 1e-4.
"""
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


def _run(torch, name, prec, n=24):
    from paper_2604_12891_b200 import Model
    c = inputs.config(name)
    d = c["dims"].replace(n_layer=1, precision=prec)
    w = inputs.make_weights(d, c["seed"])
    f, l = inputs.make_features(d, n, c["seed"] + 3, workload="large")
    m = Model(w, d)
    ft, lt = torch.from_numpy(f).cuda(), torch.from_numpy(l).cuda()
    s = torch.empty(n, dtype=torch.float32, device="cuda")
    m.tcl_score(ft, lt, s)
    m.tcl_sync_error()
    return d, w, f, l, m, s.cpu().numpy()


def _close(got, ref, rtol, what):
    scale = np.abs(ref).max() + 1e-12
    err = np.abs(got - ref)
    bad = err > rtol * scale + rtol * np.abs(ref)
    assert not bad.any(), f"{what}: {bad.sum()} / {bad.size} out of tol; max err {err.max():.3e} (scale {scale:.3e})"
    return err.max() / scale


@pytest.mark.parametrize("name,prec", [("large", 1), ("paper", 1), ("large", 0), ("tiny", 0)])
def test_stage_parity_one_layer(torch_cuda, oracle, name, prec):
    d, w, f, l, m, scores = _run(torch_cuda, name, prec)
    P = int(l.sum())
    di, dm = d.d_inner, d.d_model
    stages = {k: [] for k in ("a", "x", "z", "u", "delta", "B", "C", "g", "h")}
    ref_scores = []
    for i in range(len(l)):
        sc, st = oracle.forward_one(d, w, f[i], int(l[i]))
        ref_scores.append(sc)
        for k in stages:
            stages[k].append(st[f"layer0.{k}"])
    ref = {k: np.concatenate(v, 0) for k, v in stages.items()}
    h_enc = np.concatenate([oracle.forward_one(d, w, f[i], int(l[i]))[1]["h_enc"] for i in range(len(l))], 0)
    rtol = 2e-2 if prec == 1 else 1e-4
    A = m.debug_read("A", P, dm)
    G = m.debug_read("G", P, di)
    H = m.debug_read("H", P, dm)
    rep = {}
    lnf_path = prec == 1 and dm >= 128
    if lnf_path:
        # bf16 path: the last layer's epilogue writes LN_f(h) (the head's input) into A and leaves
        # H at its pre-layer value (the encoder output for a 1-layer model)
        W = inputs.split_weights(d, w)
        lnf = oracle.layernorm(ref["h"], W["lnf_w"], W["lnf_b"], d.ln_eps)
        rep["A"] = _close(A, lnf, rtol, "LN_f(h)")
        rep["h_enc"] = _close(H, h_enc, rtol, "encoder output")
    else:
        rep["A"] = _close(A, ref["a"], rtol, "LN_0(H_enc)")
    if prec == 1:
        # bf16 path: the fused in_proj + mixer-prep kernel (inmix.cu) keeps x on chip and stores the
        # mixer's gate SiLU(z) (the scan reads it as is)
        zr = ref["z"]
        rep["z"] = _close(m.debug_read("GZ", P, di), zr / (1.0 + np.exp(-zr)), rtol, "in_proj SiLU(z)")
    else:
        XZ = m.debug_read("XZ", P, 2 * di)
        rep["x"] = _close(XZ[:, :di], ref["x"], rtol, "in_proj x")
        rep["z"] = _close(XZ[:, di:], ref["z"], rtol, "in_proj z")
    # the mixer's intermediates: conv + SiLU output u, Delta = softplus(dt_proj), x_proj's B and C
    if prec == 1:   # (the fp32 path's fused mixer keeps them on chip)
        U = m.debug_read("U", P, di)
        DL = m.debug_read("DELTA", P, di)
        rep["u"] = _close(U, ref["u"], rtol, "conv + SiLU u")
        rep["delta"] = _close(DL, ref["delta"], rtol, "Delta")
        BC = m.debug_read("BC", P, 2 * d.d_state)
        rep["B"] = _close(BC[:, :d.d_state], ref["B"], rtol, "B")
        rep["C"] = _close(BC[:, d.d_state:], ref["C"], rtol, "C")
    rep["g"] = _close(G, ref["g"], rtol, "gated scan output")
    if not lnf_path:
        rep["h"] = _close(H, ref["h"], rtol, "residual after layer 0")
    ref_scores = np.array(ref_scores)
    rep["score"] = float(np.abs(scores - ref_scores).max())
    assert np.all(np.abs(scores - ref_scores) <= rtol * np.maximum(1, np.abs(ref_scores)))
    print(name, "prec", prec, {k: f"{v:.2e}" for k, v in rep.items()})


def _seam_lens(L, n_tiles=8, stride=125):
    """Lengths whose candidate starts fall on every row 125 m + d, d in -3..3, for m = 1..n_tiles (the
    row-tile seams of k_inconv: tile m covers rows [125 m - 3, 125 m + 125), its first 3 rows being the
    conv halo) and around its 16-row conv groups, with filler candidates of length <= L in between:
    lengths 1, 2, 3 at the seams, and candidates that start in one tile's halo and end in the next."""
    starts = {0}
    for m in range(1, n_tiles + 1):
        starts.update(stride * m + d for d in range(-3, 4))
    # ... and around the 16-row conv groups inside the tiles (a group's 3 halo rows are the rows
    # before it): tile-local rows 16 k + d, d in -2..1, in every other tile
    for m in range(0, n_tiles + 1, 2):
        for k in range(1, 8):
            starts.update(stride * m - 3 + 16 * k + d for d in range(-2, 2))
    end = stride * (n_tiles + 1)
    pos = sorted(starts)
    full = [pos[0]]
    for a in pos[1:] + [end]:
        while a - full[-1] > L:
            full.append(full[-1] + min(L, 37))   # fillers (37: not a divisor of the stride)
        full.append(a)
    return np.diff(np.array(full)).astype(np.int32)


@pytest.mark.parametrize("name", ["large", "paper", "tiny"])
def test_inconv_tile_seams_bf16(torch_cuda, oracle, name):
    """k_inconv's conv halo at the row-tile seams: u, Delta, B, C and SiLU(z) of every row of a
    1-layer bf16 model against the oracle's stage dumps, with candidate starts placed on each of the
    7 rows around every seam (d_inner 256: 2-CTA cluster; 128; 64)."""
    from paper_2604_12891_b200 import Model
    c = inputs.config(name)
    d = c["dims"].replace(n_layer=1, precision=1)
    w = inputs.make_weights(d, c["seed"])
    lens = _seam_lens(d.max_len)
    n = len(lens)
    f, _ = inputs.make_features(d, n, c["seed"] + 5, workload="large")
    m = Model(w, d)
    ft, lt = torch_cuda.from_numpy(f).cuda(), torch_cuda.from_numpy(lens).cuda()
    s = torch_cuda.empty(n, dtype=torch_cuda.float32, device="cuda")
    m.tcl_score(ft, lt, s)
    m.tcl_sync_error()
    P = int(lens.sum())
    di = d.d_inner
    ref = {k: [] for k in ("u", "delta", "B", "C", "z")}
    for i in range(n):
        _, st = oracle.forward_one(d, w, f[i], int(lens[i]))
        for k in ref:
            ref[k].append(st[f"layer0.{k}"])
    ref = {k: np.concatenate(v, 0) for k, v in ref.items()}
    rtol = 2e-2
    _close(m.debug_read("U", P, di), ref["u"], rtol, "conv + SiLU u")
    _close(m.debug_read("DELTA", P, di), ref["delta"], rtol, "Delta")
    BC = m.debug_read("BC", P, 2 * d.d_state)
    _close(BC[:, :d.d_state], ref["B"], rtol, "B")
    _close(BC[:, d.d_state:], ref["C"], rtol, "C")
    zr = ref["z"]
    _close(m.debug_read("GZ", P, di), zr / (1.0 + np.exp(-zr)), rtol, "SiLU(z)")
