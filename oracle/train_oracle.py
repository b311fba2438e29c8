"""fp64 CPU oracle of the training step: the cost model's forward in plain
PyTorch fp64 ops, the LambdaRank loss of PAPER.md Eq. 6, parameter gradients by autograd, Adam.

TEST INFRASTRUCTURE ONLY: only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
`--impl reference` legs may import this module.  The product path never imports it.

The forward follows PAPER.md §5.2 in the same step order (and readings R1-R17) as the C oracle
(oracle/tcl_oracle.c, which it is pinned against to 1e-12 in tests/test_train_pins.py); the scan
is the plain sequential recurrence (Eqs. 4-5, ZOH per R5).  Gradients are autograd's, pinned
against central finite differences of the C oracle.  The loss (reading R24):

    L = mean over groups g of  sum_{i,j in g, y_i > y_j} dNDCG(i,j) log2(1 + exp(-sigma (s_i - s_j)))
    dNDCG(i,j) = |G_i - G_j| |1/D_i - 1/D_j|,  G_i = (2^{y_i} - 1) / maxDCG,  D_i = log2(1 + rank_i)
    y_i = min latency of the group / latency_i (relevance in (0, 1]), rank_i = 1-based position of i
    when the group is sorted by predicted score (desc; ties: lower index first), maxDCG = the DCG of
    the ideal ordering (by y desc): sum_r (2^{y_(r)} - 1) / log2(1 + r).

Eq. 6's leading minus sign is read as a typesetting slip (the pair term is positive and the loss
is minimised).  Ranks, G and D are piecewise constant in the scores, so autograd
differentiates only the logistic pair term -- the LambdaRank gradient.
"""
from __future__ import annotations

import math
from typing import Dict, Tuple

import numpy as np
import torch

import inputs

F64 = torch.float64


def params_from_blob(d, blob: np.ndarray) -> Dict[str, torch.Tensor]:
    """fp64 leaf tensors (requires_grad) named as in the canonical blob (include/tcl.h)."""
    return {k: torch.tensor(v.astype(np.float64), dtype=F64, requires_grad=True) for k, v in inputs.split_weights(d, blob).items()}


def grads_to_blob(d, P: Dict[str, torch.Tensor]) -> np.ndarray:
    parts = []
    for name, shp in inputs.weight_layout(d):
        g = P[name].grad
        parts.append((g if g is not None else torch.zeros(shp, dtype=F64)).detach().numpy().ravel())
    return np.concatenate(parts)


def _silu(v):
    return v * torch.sigmoid(v)


def _layernorm(x, g, b, eps):
    mu = x.mean(-1, keepdim=True)
    var = ((x - mu) ** 2).mean(-1, keepdim=True)     # biased variance (R2)
    return (x - mu) / torch.sqrt(var + eps) * g + b


def forward_one(d, P, x: torch.Tensor) -> torch.Tensor:
    """Score of one candidate, x [T, d_in] (its T real tokens)."""
    T = x.shape[0]
    di, N, R = d.d_inner, d.d_state, d.dt_rank
    # encoder (R1)
    h = _silu(x @ P["enc.W1"].T + P["enc.b1"])
    h = _silu(h @ P["enc.W2"].T + P["enc.b2"])
    h = h @ P["enc.W3"].T + P["enc.b3"]
    for l in range(d.n_layer):
        p = f"layer{l}."
        a = _layernorm(h, P[p + "ln_w"], P[p + "ln_b"], d.ln_eps)          # pre-norm (R3)
        xz = a @ P[p + "W_in"].T                                            # in_proj, no bias
        xs, z = xz[:, :di], xz[:, di:]
        # causal depthwise conv (taps w[k] on x[t - (dc-1) + k]) + SiLU (R4)
        dc = d.d_conv
        xp = torch.cat([torch.zeros(dc - 1, di, dtype=F64), xs], 0)
        pre = P[p + "b_conv"] + sum(P[p + "w_conv"][:, k] * xp[k:k + T] for k in range(dc))
        u = _silu(pre)
        dbc = u @ P[p + "W_x"].T                                            # x_proj (R7)
        dtr, Bm, Cm = dbc[:, :R], dbc[:, R:R + N], dbc[:, R + N:]
        delta = torch.nn.functional.softplus(dtr @ P[p + "W_dt"].T + P[p + "b_dt"])
        A = -torch.exp(P[p + "A_log"])                                      # R8
        s = torch.zeros(di, N, dtype=F64)
        ys = []
        for t in range(T):                                                  # Eqs. 4-5, ZOH (R5)
            dA = delta[t][:, None] * A
            Ab = torch.exp(dA)
            if d.disc == inputs.DISC_ZOH:
                Bb = (Ab - 1.0) / A * Bm[t][None, :]
            else:
                Bb = delta[t][:, None] * Bm[t][None, :]
            s = Ab * s + Bb * u[t][:, None]
            ys.append(s @ Cm[t] + P[p + "Dv"] * u[t])
        y = torch.stack(ys, 0)
        g = y * _silu(z)
        h = h + g @ P[p + "W_out"].T                                        # out_proj + residual
    f = _layernorm(h, P["lnf_w"], P["lnf_b"], d.ln_eps)
    pooled = f.mean(0)                                                      # masked mean (R9)
    q = _silu(pooled @ P["dec.W1"].T + P["dec.b1"])
    q = _silu(q @ P["dec.W2"].T + P["dec.b2"])
    return (q @ P["dec.W3"].T + P["dec.b3"])[0]


def forward(d, P, feats: np.ndarray, lens: np.ndarray) -> torch.Tensor:
    return torch.stack([forward_one(d, P, torch.tensor(feats[i, :int(lens[i])].astype(np.float64), dtype=F64))
                        for i in range(len(lens))])


def relevance(latency: np.ndarray, offsets: np.ndarray) -> np.ndarray:
    """y_i = min latency of i's group / latency_i (reading R24)."""
    y = np.empty(latency.shape[0], np.float64)
    for g in range(len(offsets) - 1):
        a, b = offsets[g], offsets[g + 1]
        lat = latency[a:b].astype(np.float64)
        y[a:b] = lat.min() / lat
    return y


def lambdarank_loss(scores: torch.Tensor, latency: np.ndarray, offsets: np.ndarray, sigma: float = 1.0) -> torch.Tensor:
    """Eq. 6 (reading R24), averaged over the groups."""
    y_all = relevance(latency, offsets)
    total = torch.zeros((), dtype=F64)
    n_groups = len(offsets) - 1
    for g in range(n_groups):
        a, b = int(offsets[g]), int(offsets[g + 1])
        s = scores[a:b]
        y = y_all[a:b]
        n = b - a
        sv = s.detach().numpy()
        order = sorted(range(n), key=lambda i: (-sv[i], i))                 # rank by predicted score
        rank = np.empty(n, np.int64)
        for r, i in enumerate(order):
            rank[i] = r + 1
        gain = 2.0 ** y - 1.0
        ideal = sorted(gain, reverse=True)
        max_dcg = sum(gv / math.log2(1 + r + 1) for r, gv in enumerate(ideal))
        G = gain / max_dcg
        D = np.log2(1.0 + rank)
        # all ordered pairs (i, j) with y_i > y_j, as matrices indexed [i, j]
        pair = y[:, None] > y[None, :]
        dndcg = np.abs(G[:, None] - G[None, :]) * np.abs(1.0 / D[:, None] - 1.0 / D[None, :])
        # log2(1 + e^-x) written as softplus(-x) / ln 2 (the same function, no overflow for large |x|)
        term = torch.nn.functional.softplus(-sigma * (s[:, None] - s[None, :])) / math.log(2.0)
        w = torch.tensor(np.where(pair, dndcg, 0.0), dtype=F64)
        total = total + torch.where(torch.tensor(pair), w * term, torch.zeros((), dtype=F64)).sum()
    return total / n_groups


def train_grads(d, blob: np.ndarray, feats, lens, latency, offsets, sigma: float = 1.0
                ) -> Tuple[float, np.ndarray, np.ndarray, np.ndarray]:
    """(loss, grad blob [canonical layout], scores, dL/dscores) of one training batch."""
    P = params_from_blob(d, blob)
    s = forward(d, P, feats, lens)
    s.retain_grad()
    loss = lambdarank_loss(s, latency, offsets, sigma)
    loss.backward()
    return float(loss.detach()), grads_to_blob(d, P), s.detach().numpy(), s.grad.numpy()


def loss_and_score_grad(scores: np.ndarray, latency, offsets, sigma: float = 1.0) -> Tuple[float, np.ndarray]:
    s = torch.tensor(scores.astype(np.float64), dtype=F64, requires_grad=True)
    loss = lambdarank_loss(s, latency, offsets, sigma)
    loss.backward()
    return float(loss.detach()), s.grad.numpy()


def adam_step(w, g, m, v, t: int, lr: float, b1: float = 0.9, b2: float = 0.999, eps: float = 1e-8):
    """One Adam update (Kingma & Ba, Alg. 1) in fp64; t is the 1-based step.  Returns (w, m, v)."""
    m = b1 * m + (1 - b1) * g
    v = b2 * v + (1 - b2) * g * g
    mh = m / (1 - b1 ** t)
    vh = v / (1 - b2 ** t)
    return w - lr * mh / (np.sqrt(vh) + eps), m, v
