"""GPU parity of the training step (tcl_train_step; Eq. 6 LambdaRank, backward, Adam; reading R24)
against oracle/train_oracle.py (fp64 autograd).

Tolerances (derived in DESIGN.md R24): loss 1e-4 relative; dL/dscore and every weight gradient
within 1e-3 of the largest |gradient| of its tensor (fp32 forward/backward accumulation over at
most a few thousand rows); Adam applied to the GPU's own gradients within 1e-6 relative.
The ranking inside each group is an integer decision taken on fp32 scores: the test checks that
GPU and oracle scores order every group identically (the seeds keep pairs apart).
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


def _batch(name, n, group, seed=0):
    c = inputs.config(name)
    d = c["dims"]
    w = inputs.make_weights(d, c["seed"])
    f, l = inputs.make_features(d, n, c["seed"] + 1 + seed, workload="tuning")
    rng = np.random.default_rng(100 + seed)
    lat = np.exp(rng.normal(-6.0, 0.7, n)).astype(np.float32)
    off = np.arange(0, n + 1, group, dtype=np.int64)
    if off[-1] != n:
        off = np.r_[off, n]
    return d, w, f, l, lat, off


def _dev(torch, *arrs):
    return [torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in arrs]


@pytest.mark.parametrize("name,n,group", [("tiny", 48, 12), ("tuning", 40, 20), ("paper", 37, 9)])
def test_train_step_gradients(torch_cuda, name, n, group):
    from oracle import train_oracle as TO
    from paper_2604_12891_b200 import Model
    d, w, f, l, lat, off = _batch(name, n, group)
    m = Model(w, d)
    m.tcl_train_init(n)
    ft, lt, latt, offt = _dev(torch_cuda, f, l, lat, off)
    loss = torch_cuda.zeros(1, device="cuda")
    m.tcl_train_step(ft, lt, latt, offt, int(np.diff(off).max()), apply_update=False, loss=loss)
    m.tcl_sync_error()
    ref_loss, ref_g, ref_s, ref_ds = TO.train_grads(d, w, f, l, lat, off)
    s = m.tcl_train_read("scores", n)
    for gi in range(len(off) - 1):
        a, b = off[gi], off[gi + 1]
        assert np.argsort(-s[a:b], kind="stable").tolist() == np.argsort(-ref_s[a:b], kind="stable").tolist()
    assert float(loss.item()) == pytest.approx(ref_loss, rel=1e-4)
    ds = m.tcl_train_read("dscores", n)
    assert np.abs(ds - ref_ds).max() <= 1e-3 * np.abs(ref_ds).max()
    g = m.tcl_train_read("grads", inputs.weights_count(d))
    gmax = np.abs(ref_g).max()
    # dec.b3's gradient is the plain fp32 sum of the n dscores, whose exact value is 0 (antisymmetric
    # pair lambdas): its error is bounded by the dscores' own errors plus the summation error of n
    # fp32 additions, n 2^-24 sum |ds| (standard recursive-summation bound)
    b3_floor = np.abs(ds - ref_ds).sum() + n * 2.0 ** -24 * np.abs(ds).sum()
    for ent in inputs.manifest(d):
        o, cnt = ent["offset"], int(np.prod(ent["shape"]))
        ref = ref_g[o:o + cnt]
        err = np.abs(g[o:o + cnt] - ref).max()
        # + 1e-6 of the global scale: tensors whose exact gradient vanishes carry only fp32
        # cancellation residue
        floor = max(1e-6 * gmax, b3_floor if ent["name"] == "dec.b3" else 0.0)
        assert err <= 1e-3 * np.abs(ref).max() + floor, (ent["name"], err, np.abs(ref).max(), floor)
    # the model is unchanged without apply_update
    assert np.array_equal(m.tcl_train_read("weights", w.size), w)


def test_adam_update_and_refresh(torch_cuda, oracle):
    from oracle import train_oracle as TO
    from paper_2604_12891_b200 import Model
    d, w, f, l, lat, off = _batch("tiny", 32, 16, seed=1)
    m = Model(w, d)
    lr = 1e-3
    m.tcl_train_init(32, lr=lr)
    ft, lt, latt, offt = _dev(torch_cuda, f, l, lat, off)
    m.tcl_train_step(ft, lt, latt, offt, 16, apply_update=True)
    m.tcl_sync_error()
    g = m.tcl_train_read("grads", w.size).astype(np.float64)
    w1 = m.tcl_train_read("weights", w.size).astype(np.float64)
    ref, _, _ = TO.adam_step(w.astype(np.float64), g, np.zeros(w.size), np.zeros(w.size), 1, lr)
    assert np.abs(w1 - ref).max() <= 1e-6 * np.abs(ref).max() + 1e-3 * lr
    # scoring now uses the updated weights (derived copies refreshed): equals a fresh model of w1
    s_trained = torch_cuda.empty(32, device="cuda")
    m.tcl_score(ft, lt, s_trained)
    fresh = Model(w1.astype(np.float32), d)
    s_fresh = torch_cuda.empty(32, device="cuda")
    fresh.tcl_score(ft, lt, s_fresh)
    assert np.array_equal(s_trained.cpu().numpy(), s_fresh.cpu().numpy())


def test_training_reduces_the_loss(torch_cuda):
    from paper_2604_12891_b200 import Model
    d, w, f, l, lat, off = _batch("tuning", 256, 64, seed=2)
    m = Model(w, d)
    m.tcl_train_init(256, lr=2e-3)
    ft, lt, latt, offt = _dev(torch_cuda, f, l, lat, off)
    loss = torch_cuda.zeros(1, device="cuda")
    hist = []
    for _ in range(30):
        m.tcl_train_step(ft, lt, latt, offt, 64, apply_update=True, loss=loss)
        hist.append(float(loss.item()))
    assert np.isfinite(hist).all()
    assert hist[-1] < 0.8 * hist[0], hist


def test_train_errors(torch_cuda):
    from paper_2604_12891_b200 import Model
    from paper_2604_12891_b200.tcl import TclError
    d, w, f, l, lat, off = _batch("tiny", 16, 8)
    m = Model(w, d)
    ft, lt, latt, offt = _dev(torch_cuda, f, l, lat, off)
    with pytest.raises(TclError):
        m.tcl_train_step(ft, lt, latt, offt, 8)          # no tcl_train_init
    c = inputs.config("large")
    with pytest.raises(TclError):
        Model(inputs.make_weights(c["dims"], 1), c["dims"]).tcl_train_init(16)


_STEPS_SCRIPT = r'''
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
import inputs
from paper_2604_12891_b200 import Model
c = inputs.config("tiny"); d = c["dims"]
w = inputs.make_weights(d, c["seed"])
f, l = inputs.make_features(d, 32, 7, workload="tuning")
lat = np.exp(np.random.default_rng(3).normal(-6, 0.7, 32)).astype(np.float32)
off = np.arange(0, 33, 8, dtype=np.int64)
m = Model(w, d)
m.use_graphs(sys.argv[3] == "1")
m.tcl_train_init(32, lr=1e-3)
ft, lt, latt, offt = (torch.from_numpy(a).cuda() for a in (f, l, lat, off))
loss = torch.zeros(1, device="cuda")
for _ in range(3):
    m.tcl_train_step(ft, lt, latt, offt, 8, True, loss)
# Alg. 1 loop: score a pool much larger than the training batch (the workspace grows and is
# reallocated), then train again -- a replayed step graph must not use the freed buffers
fp, lp = inputs.make_features(d, 20000, 8, workload="tuning")
sp = torch.empty(20000, device="cuda")
m.tcl_score(torch.from_numpy(fp).cuda(), torch.from_numpy(lp).cuda(), sp)
for _ in range(2):
    m.tcl_train_step(ft, lt, latt, offt, 8, True, loss)
m.tcl_sync_error()
np.save(sys.argv[2], np.concatenate([m.tcl_train_read("weights", w.size), sp.cpu().numpy()]))
'''


def test_graph_replay_equals_direct_launches(torch_cuda, tmp_path):
    '''The captured step graph (default) and direct launches (TCL_OPT_GRAPHS = 0) give bit-identical
    weights after 3 Adam steps, a pool scoring that reallocates the workspace, and 2 more steps
    (the step counter and bias corrections live on the device; the graph is re-captured when the
    workspace it baked in is reallocated).'''
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    script = tmp_path / "steps.py"
    script.write_text(_STEPS_SCRIPT)
    out = {}
    for mode in ("1", "0"):
        path = tmp_path / f"w{mode}.npy"
        subprocess.run([sys.executable, str(script), root, str(path), mode], check=True, timeout=300)
        out[mode] = np.load(path)
    assert np.isfinite(out["0"]).all()
    assert np.array_equal(out["1"], out["0"])


def test_bad_groups_flagged(torch_cuda):
    '''A group larger than max_group (or with < 2 members) is skipped and flagged (TCL_ESHAPE);
    candidates outside every group get a zero score gradient.'''
    from paper_2604_12891_b200 import Model, TclError
    c = inputs.config("tiny")
    d = c["dims"]
    w = inputs.make_weights(d, c["seed"])
    f, l = inputs.make_features(d, 32, 7, workload="tuning")
    lat = np.exp(np.random.default_rng(3).normal(-6, 0.7, 32)).astype(np.float32)
    m = Model(w, d)
    m.tcl_train_init(32)
    off = np.array([0, 8, 24, 30], dtype=np.int64)      # group 1 has 16 > max_group = 8; 30..31 uncovered
    ft, lt, latt, offt = _dev(torch_cuda, f, l, lat, off)
    m.tcl_train_step(ft, lt, latt, offt, 8, False)
    with pytest.raises(TclError) as e:
        m.tcl_sync_error()
    assert e.value.code == -2
    ds = m.tcl_train_read("dscores", 32)
    assert np.all(ds[8:24] == 0) and np.all(ds[30:] == 0) and np.any(ds[:8] != 0)
