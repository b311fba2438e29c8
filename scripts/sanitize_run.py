"""One small invocation of every kernel family, for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck): fp32 path (tiny: SIMT + 3xTF32 GEMMs, fp32 mixer, both scan modes),
bf16 path (tiny d_model 64, tuning d_model 128 and large at n = 64: tcgen05 GEMMs with TMA, k_inconv
(2-CTA cluster at large), k_xdt, scan, encoder),
MC dropout, top-k (radix + bitonic), the multi-GPU key halves, RDU selection, Top-k score, one
training step.  Graph replay is off so every launch is a plain kernel launch."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import inputs  # noqa: E402
from paper_2604_12891_b200 import Model  # noqa: E402


def dev(*a):
    return [torch.from_numpy(np.ascontiguousarray(x)).cuda() for x in a]


def run(name, prec, n, scan=None):
    c = inputs.config(name)
    d = c["dims"].replace(precision=prec)
    m = Model(inputs.make_weights(d, c["seed"]), d)
    m.use_graphs(False)
    if scan:
        m.scan_mode(scan)
    f, l = inputs.make_features(d, n, c["seed"] + 1, workload="large" if name == "large" else "tuning")
    ft, lt = dev(f, l)
    s = torch.empty(n, device="cuda")
    m.tcl_score(ft, lt, s)
    mean, var = torch.empty(n, device="cuda"), torch.empty(n, device="cuda")
    m.tcl_score_mc(ft, lt, 2, 7, 0, mean, var)
    for k in (8, 300 if n >= 300 else 16, 1500):
        idx, top = torch.empty(k, dtype=torch.int64, device="cuda"), torch.empty(k, device="cuda")
        m.tcl_topk(s, k, 0, idx, top)
    keys = torch.empty(16, dtype=torch.int64, device="cuda")
    m.tcl_topk_local_keys(s, 0, 16, keys)
    idx, top = torch.empty(16, dtype=torch.int64, device="cuda"), torch.empty(16, device="cuda")
    m.tcl_topk_merge_keys(keys, 16, idx, top)
    m.tcl_sync_error()
    print(name, prec, scan, "ok", float(s.sum()))
    return m, d, ft, lt


run("tiny", 0, 200)
run("tiny", 0, 200, scan="chunked")
run("tiny", 1, 200)
run("tuning", 1, 300)
run("large", 1, 64)
m, d, ft, lt = run("paper", 0, 256)
# RDU selection + Top-k score
pool = torch.randn(3000, device="cuda")
ops = torch.randint(0, 5, (3000,), dtype=torch.int32, device="cuda")
lab = torch.randn(50, device="cuda")
sel = torch.empty(100, dtype=torch.int64, device="cuda")
ns = torch.empty(1, dtype=torch.int32, device="cuda")
m.tcl_rdu_select(pool, ops, lab, 5, 100, sel, ns)
off = torch.tensor([0, 100, 250, 256], dtype=torch.int64, device="cuda")
lat = torch.rand(256, device="cuda") + 0.1
res = torch.empty(3, dtype=torch.float64, device="cuda")
s = torch.empty(256, device="cuda")
m.tcl_score(ft, lt, s)
m.tcl_topk_score(s, lat, off, torch.ones(3, device="cuda"), 256, [5], res)
# one training step (tiny)
c = inputs.config("tiny")
dt = c["dims"]
mt = Model(inputs.make_weights(dt, c["seed"]), dt)
mt.use_graphs(False)
f, l = inputs.make_features(dt, 32, 5, workload="tuning")
lat = np.exp(np.random.default_rng(3).normal(-6, 0.7, 32)).astype(np.float32)
offs = np.arange(0, 33, 8, dtype=np.int64)
mt.tcl_train_init(32)
ft2, lt2, lat2, off2 = dev(f, l, lat, offs)
mt.tcl_train_step(ft2, lt2, lat2, off2, 8, True)
mt.tcl_sync_error()
torch.cuda.synchronize()
print("all ok")
