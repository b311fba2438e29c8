"""Seeded synthetic inputs shared by the oracle tests, the GPU tests and bench.py.

This module holds NO arithmetic of the method (no layer, no scan, no score):
it only draws random numbers.  Both sides of every parity check -- the fp64 CPU
oracle (`oracle/`) and the CUDA path (`paper_2604_12891_b200/`) -- read the
weights blob and feature tensors this module produces; neither imports the other.

Contents
  * CONFIGS              -- the six configurations of SURVEY.md §8.0 (tiny, tuning,
                            rdu, large, long, paper).  Readings R10/R11 fill the
                            silent entries: encoder widths [dm/2, dm, dm], decoder
                            widths [dm/2, dm/4, 1] (reproduce PAPER.md:451's
                            64/128/128 and 64/32/1 at d_model=128), dt_rank =
                            ceil(dm/16), D = 22 (CPU feature width).
  * weight_layout(dims)  -- names/shapes of the canonical fp32 blob.
  * make_weights(dims, seed) -- reading R20 (seeded random init).
  * make_features(dims, n, seed, ...) -- Tenset-style synthetic schedule-feature
                            sequences (SPEC.md:152-170 token recipe).
"""
from __future__ import annotations

import dataclasses
import math
from typing import Dict, List, Tuple

import numpy as np

PREC_FP32 = 0
PREC_BF16_PROJ = 1
DISC_ZOH = 0
DISC_EULER_B = 1


@dataclasses.dataclass
class Dims:
    """Mirrors `tcl_dims` of include/tcl.h field for field (same order, same types)."""
    d_in: int = 22
    max_len: int = 25
    d_model: int = 64
    n_layer: int = 1
    d_state: int = 16
    d_conv: int = 4
    expand: int = 1
    dt_rank: int = 4
    enc_dims: Tuple[int, int, int] = (32, 64, 64)
    dec_dims: Tuple[int, int, int] = (32, 16, 1)
    ln_eps: float = 1e-5
    dropout_p: float = 0.1
    precision: int = PREC_FP32
    disc: int = DISC_ZOH

    @property
    def d_inner(self) -> int:
        return self.expand * self.d_model

    def replace(self, **kw) -> "Dims":
        return dataclasses.replace(self, **kw)


def _dims_for(n_layer: int, dm: int, d_state: int, max_len: int, precision: int,
              expand: int = 1, d_conv: int = 4, d_in: int = 22) -> Dims:
    return Dims(d_in=d_in, max_len=max_len, d_model=dm, n_layer=n_layer, d_state=d_state,
                d_conv=d_conv, expand=expand, dt_rank=int(math.ceil(dm / 16)),
                enc_dims=(dm // 2, dm, dm), dec_dims=(dm // 2, dm // 4, 1),
                ln_eps=1e-5, dropout_p=0.1, precision=precision, disc=DISC_ZOH)


# SURVEY.md §8.0 config table.  `n` = candidates on one GPU (per rank under weak scaling).
CONFIGS: Dict[str, dict] = {
    "tiny":   dict(dims=_dims_for(1, 64, 16, 25, PREC_FP32), n=256, topk=16, mc_passes=0, seed=1000),
    "tuning": dict(dims=_dims_for(2, 128, 8, 25, PREC_FP32), n=4096, topk=64, mc_passes=0, seed=1001),
    "rdu":    dict(dims=_dims_for(2, 128, 8, 25, PREC_FP32), n=16384, topk=0, mc_passes=10, seed=1002),
    "large":  dict(dims=_dims_for(4, 256, 16, 64, PREC_BF16_PROJ), n=65536, topk=64, mc_passes=0, seed=1003),
    "long":   dict(dims=_dims_for(4, 256, 16, 128, PREC_BF16_PROJ), n=1048576, topk=1024, mc_passes=0, seed=1004),
    # Paper reference model [n_layer, d_state, expand, d_conv] = [1, 8, 1, 4],
    # d_model 128, CPU features 26x22.
    "paper":  dict(dims=_dims_for(1, 128, 8, 26, PREC_FP32), n=1024, topk=16, mc_passes=0, seed=1005),
}


def weight_layout(d: Dims) -> List[Tuple[str, Tuple[int, ...]]]:
    """Canonical blob order; PyTorch [out, in] row-major."""
    e1, e2, e3 = d.enc_dims
    h1, h2, h3 = d.dec_dims
    di, N, R, dm = d.d_inner, d.d_state, d.dt_rank, d.d_model
    out: List[Tuple[str, Tuple[int, ...]]] = [
        ("enc.W1", (e1, d.d_in)), ("enc.b1", (e1,)),
        ("enc.W2", (e2, e1)), ("enc.b2", (e2,)),
        ("enc.W3", (e3, e2)), ("enc.b3", (e3,)),
    ]
    for l in range(d.n_layer):
        p = f"layer{l}."
        out += [
            (p + "ln_w", (dm,)), (p + "ln_b", (dm,)),
            (p + "W_in", (2 * di, dm)),
            (p + "w_conv", (di, d.d_conv)), (p + "b_conv", (di,)),
            (p + "W_x", (R + 2 * N, di)),
            (p + "W_dt", (di, R)), (p + "b_dt", (di,)),
            (p + "A_log", (di, N)), (p + "Dv", (di,)),
            (p + "W_out", (dm, di)),
        ]
    out += [("lnf_w", (dm,)), ("lnf_b", (dm,)),
            ("dec.W1", (h1, dm)), ("dec.b1", (h1,)),
            ("dec.W2", (h2, h1)), ("dec.b2", (h2,)),
            ("dec.W3", (h3, h2)), ("dec.b3", (h3,))]
    return out


def weights_count(d: Dims) -> int:
    return int(sum(int(np.prod(s)) for _, s in weight_layout(d)))


def manifest(d: Dims) -> List[dict]:
    """SPEC-style manifest: name, shape, offset (in floats)."""
    off, out = 0, []
    for name, shape in weight_layout(d):
        cnt = int(np.prod(shape))
        out.append(dict(name=name, shape=list(shape), offset=off))
        off += cnt
    return out


def split_weights(d: Dims, blob: np.ndarray) -> Dict[str, np.ndarray]:
    """View a flat blob as named arrays (no arithmetic)."""
    off, out = 0, {}
    for name, shape in weight_layout(d):
        cnt = int(np.prod(shape))
        out[name] = blob[off:off + cnt].reshape(shape)
        off += cnt
    assert off == blob.size
    return out


def make_weights(d: Dims, seed: int) -> np.ndarray:
    """Reading R20: PCG64-seeded random init of every tensor, fp32 blob."""
    rng = np.random.Generator(np.random.PCG64(seed))
    parts = []
    for name, shape in weight_layout(d):
        base = name.split(".")[-1]
        if base.startswith("W") and base not in ("W_dt",):
            fan_in = shape[1]
            # LeCun-uniform bound sqrt(3/fan_in): unit-variance-preserving, so every stage
            # carries O(1) signal and scores spread well beyond the parity tolerance.
            v = rng.uniform(-1.0, 1.0, shape) * math.sqrt(3.0 / fan_in)
        elif base in ("b1", "b2", "b3"):
            # bias of the preceding linear: same fan-in bound
            prev_w = [s for nm, s in weight_layout(d) if nm == name[:-2] + "W" + base[1]][0]
            v = rng.uniform(-1.0, 1.0, shape) / math.sqrt(prev_w[1])
        elif base == "w_conv":
            v = rng.uniform(-1.0, 1.0, shape) / math.sqrt(d.d_conv)
        elif base == "b_conv":
            v = rng.uniform(-1.0, 1.0, shape) / math.sqrt(d.d_conv)
        elif base == "W_dt":
            v = rng.uniform(-1.0, 1.0, shape) / math.sqrt(d.dt_rank)
        elif base == "b_dt":
            dt = np.exp(rng.uniform(math.log(1e-3), math.log(1e-1), shape))
            v = np.log(np.expm1(dt))          # inverse softplus of the drawn step size
        elif base == "A_log":
            v = np.log(np.arange(1, d.d_state + 1, dtype=np.float64))[None, :] \
                + rng.uniform(-0.5, 0.5, shape)
        elif base == "Dv":
            v = rng.uniform(0.5, 1.5, shape)
        elif base in ("ln_w", "lnf_w"):
            v = rng.uniform(0.8, 1.2, shape)
        elif base in ("ln_b", "lnf_b"):
            v = rng.uniform(-0.1, 0.1, shape)
        else:  # pragma: no cover
            raise KeyError(name)
        parts.append(np.asarray(v, dtype=np.float32).ravel())
    blob = np.concatenate(parts)
    assert blob.size == weights_count(d)
    return blob


# ---------------------------------------------------------------------------------------
# Tenset-style synthetic schedule-feature sequences.
# Token t of a real candidate = [one-hot(kind) over SPEC's 10 primitive kinds (cols 0-9),
# log1p(param) (col 10), platform vector (cols 11-21)]; padded rows trail.
N_KINDS = 10
OP_EXTENTS = {  # loop extents per SPEC operator type; values only seed parameter draws
    "conv2d": [1, 64, 56, 56, 64, 3, 3], "conv3d": [1, 32, 16, 28, 28, 32, 3],
    "matmul": [1, 512, 768, 768], "depthwise_conv": [1, 128, 112, 112, 3, 3],
    "pooling": [1, 64, 112, 112, 3, 3], "softmax": [1, 12, 128, 128],
    "norm": [1, 768, 128], "elementwise": [1, 256, 56, 56],
}


def _divisors(x: int) -> np.ndarray:
    return np.array([v for v in range(1, x + 1) if x % v == 0], dtype=np.int64)


def make_features(d: Dims, n: int, seed: int, workload: str = "tuning",
                  full_length: bool = False, pad_value: float = 0.0,
                  stress: bool = False, dup_frac: float = 0.01) -> Tuple[np.ndarray, np.ndarray]:
    """Return (feats float32 [n, L, D], lens int32 [n]).

    workload: "tuning" (one ResNet-50 conv2d subgraph), "rdu" (32 assignments, op skew
    0.6/0.25/0.15), "large" (64 assignments, 8 op types), "long" (512 assignments).
    pad_value: value written into padded slots (0, a float, or np.nan) -- the path must
    ignore padded slots whatever they hold (reading R16)."""
    L, D = d.max_len, d.d_in
    rng = np.random.Generator(np.random.PCG64(seed))
    hw_dim = D - (N_KINDS + 1)
    assert hw_dim >= 0
    if workload == "tuning":
        ops = ["conv2d"]
    elif workload == "rdu":
        ops = list(rng.choice(["conv2d", "matmul", "softmax"], size=32, p=[0.6, 0.25, 0.15]))
    else:
        n_as = 64 if workload == "large" else 512
        ops = list(rng.choice(list(OP_EXTENTS), size=n_as))
    n_as = len(ops)
    hw = np.clip(rng.standard_normal(hw_dim), -5, 5).astype(np.float32)

    # base schedule per assignment: L tokens of (kind, log1p(param))
    base_kind = rng.integers(0, N_KINDS, size=(n_as, L))
    base_par = np.zeros((n_as, L), dtype=np.float64)
    for a, op in enumerate(ops):
        ext = OP_EXTENTS[op]
        for t in range(L):
            e = ext[rng.integers(0, len(ext))]
            dv = _divisors(int(e))
            base_par[a, t] = dv[rng.integers(0, dv.size)]

    assign = rng.integers(0, n_as, size=n)
    lens = np.full(n, L, dtype=np.int32) if full_length else \
        rng.integers(min(4, L), L + 1, size=n).astype(np.int32)
    kind = base_kind[assign].copy()
    par = base_par[assign].copy()
    # mutations: 1-3 positions get a new kind or a new parameter (SPEC mutate_schedule S:58)
    n_mut = rng.integers(1, 4, size=n)
    for m in range(3):
        active = n_mut > m
        pos = (rng.random(n) * lens).astype(np.int64)
        what = rng.random(n) < 0.5
        rows = np.nonzero(active & what)[0]
        kind[rows, pos[rows]] = rng.integers(0, N_KINDS, size=rows.size)
        rows = np.nonzero(active & ~what)[0]
        par[rows, pos[rows]] = rng.integers(1, 225, size=rows.size)

    feats = np.zeros((n, L, D), dtype=np.float32)
    if stress:
        feats[:] = rng.standard_normal((n, L, D)).astype(np.float32)
    else:
        onehot = np.eye(N_KINDS, dtype=np.float32)[kind]        # [n, L, 10]
        feats[:, :, :N_KINDS] = onehot
        feats[:, :, N_KINDS] = np.log1p(par).astype(np.float32)
        feats[:, :, N_KINDS + 1:] = hw[None, None, :]
    # exact duplicates (ties) -- about dup_frac of the candidates copy another one
    n_dup = int(n * dup_frac)
    if n_dup > 0 and n > 1:
        dst = rng.choice(n, size=n_dup, replace=False)
        src = rng.integers(0, n, size=n_dup)
        feats[dst] = feats[src]
        lens[dst] = lens[src]
    # padded slots
    mask = np.arange(L)[None, :] >= lens[:, None]
    if isinstance(pad_value, str) and pad_value == "random":
        feats[mask] = rng.standard_normal((int(mask.sum()), D)).astype(np.float32) * 100
    else:
        feats[mask] = np.float32(pad_value)
    return feats, lens


def config(name: str) -> dict:
    c = dict(CONFIGS[name])
    c["name"] = name
    return c


def make_eval_tasks(n_tasks: int, seed: int, min_len: int = 16, max_len: int = 4096, noise: float = 0.5,
                    tie_quant: float = 0.0):
    """Synthetic evaluation tasks for the Top-k score (Eq. 12): one task per (model, subgraph).

    Shapes follow §7.1.1: a task is a subgraph with the programs measured for it (log-uniform
    count in [min_len, max_len]); latencies are log-normal around a per-task scale; the predicted
    score is a noisy monotone predictor (-log latency + noise·N(0,1)); weights are occurrence
    frequencies (integers 1..8).  tie_quant > 0 quantises the scores (forces equal scores).
    Returns (scores f32 [n], latency f32 [n], offsets i64 [n_tasks+1], weights f32 [n_tasks])."""
    rng = np.random.default_rng(seed)
    lens = np.exp(rng.uniform(np.log(min_len), np.log(max_len + 1), n_tasks)).astype(np.int64)
    lens = np.clip(lens, min_len, max_len)
    off = np.zeros(n_tasks + 1, np.int64)
    off[1:] = np.cumsum(lens)
    n = int(off[-1])
    scale = np.repeat(rng.uniform(-9.0, -3.0, n_tasks), lens)          # log-seconds per task
    lat = np.exp(scale + rng.normal(0.0, 0.6, n)).astype(np.float32)
    sc = (-np.log(lat.astype(np.float64)) + noise * rng.normal(size=n)).astype(np.float32)
    if tie_quant > 0:
        sc = (np.round(sc / tie_quant) * tie_quant).astype(np.float32)
    w = rng.integers(1, 9, n_tasks).astype(np.float32)
    return sc, lat, off, w


def adapter_layout(d: Dims, a: int) -> List[Tuple[str, Tuple[int, ...]]]:
    """KB+AC lateral adapters (Eq. 7, reading R23), per site in the order enc1, enc2, enc3,
    layer 0..n_layer-1, dec1, dec2: V [a][in], c [a], U [out][a], alpha [out]."""
    sites = [("enc1", d.d_in, d.enc_dims[0]), ("enc2", d.enc_dims[0], d.enc_dims[1]),
             ("enc3", d.enc_dims[1], d.d_model)]
    sites += [(f"layer{l}", d.d_model, d.d_model) for l in range(d.n_layer)]
    sites += [("dec1", d.d_model, d.dec_dims[0]), ("dec2", d.dec_dims[0], d.dec_dims[1])]
    out = []
    for name, i, o in sites:
        out += [(f"{name}.V", (a, i)), (f"{name}.c", (a,)), (f"{name}.U", (o, a)), (f"{name}.alpha", (o,))]
    return out


def adapters_count(d: Dims, a: int) -> int:
    return sum(int(np.prod(s)) for _, s in adapter_layout(d, a))


def make_adapters(d: Dims, a: int, seed: int, alpha_range=(0.2, 1.0)) -> np.ndarray:
    """Seeded adapter blob: V, U LeCun-uniform, c ~ U(+-1/sqrt(in)), alpha ~ U(alpha_range)."""
    rng = np.random.default_rng(seed)
    parts = []
    for name, shp in adapter_layout(d, a):
        kind = name.split(".")[1]
        if kind == "V" or kind == "U":
            fan_in = shp[1]
            v = rng.uniform(-np.sqrt(3.0 / fan_in), np.sqrt(3.0 / fan_in), shp)
        elif kind == "c":
            fan_in = [s for nm, s in adapter_layout(d, a) if nm == name.replace(".c", ".V")][0][1]
            v = rng.uniform(-1 / np.sqrt(fan_in), 1 / np.sqrt(fan_in), shp)
        else:
            v = rng.uniform(alpha_range[0], alpha_range[1], shp)
        parts.append(v.astype(np.float32).ravel())
    return np.concatenate(parts)


def split_adapters(d: Dims, a: int, blob: np.ndarray) -> Dict[str, np.ndarray]:
    out, off = {}, 0
    for name, shp in adapter_layout(d, a):
        cnt = int(np.prod(shp))
        out[name] = blob[off:off + cnt].reshape(shp)
        off += cnt
    return out


def default_adapter_rank(d: Dims) -> int:
    """Reading R23: adapter width a = dt_rank = ceil(d_model / 16) (the paper gives only the 0.7 MB
    total of KB + AC at d_model 128; a = 8 gives 0.74 MiB)."""
    return d.dt_rank
