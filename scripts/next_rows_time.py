"""Time tcl_rdu_select on the rdu configuration's pool size (and the max pool) with CUDA events."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import inputs
from paper_2604_12891_b200 import Model
c = inputs.config("tiny"); d = c["dims"]
m = Model(inputs.make_weights(d, c["seed"]), d)
sms = torch.cuda.get_device_properties(0).multi_processor_count
out = {}
for n, lab_n, B, n_ops in ((16384, 1024, 1638, 13), (131072, 4096, 4096, 40), (4096 * sms, 4096, 4096, 40)):
    rng = np.random.default_rng(0)
    pool = torch.from_numpy(rng.normal(size=n).astype(np.float32)).cuda()
    ops = torch.from_numpy(rng.integers(0, n_ops, n).astype(np.int32)).cuda()
    lab = torch.from_numpy(rng.normal(size=lab_n).astype(np.float32)).cuda()
    sel = torch.empty(B, dtype=torch.int64, device="cuda"); ns = torch.empty(1, dtype=torch.int32, device="cuda")
    for _ in range(3): m.tcl_rdu_select(pool, ops, lab, n_ops, B, sel, ns)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10): m.tcl_rdu_select(pool, ops, lab, n_ops, B, sel, ns)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    out[f"n{n}_lab{lab_n}_B{B}"] = {"ms": ms, "us_per_pick": 1000 * ms / B, "picks": int(ns.item())}
    print(n, lab_n, B, f"{ms:.3f} ms", f"{1000*ms/B:.2f} us/pick", flush=True)
json.dump(out, open("gpurun_out/next_rows_time.json", "w"), indent=1)

# Top-k score (Eq. 12): 5 models x ~ 400 subgraphs of 16..4096 programs
sc, lat, off, w = inputs.make_eval_tasks(2000, 1)
ks = [1, 5, 10]
args = [torch.from_numpy(a).cuda() for a in (sc, lat, off, w)]
res = torch.empty(9, dtype=torch.float64, device="cuda")
ml = int(np.diff(off).max())
for _ in range(3): m.tcl_topk_score(*args, ml, ks, res)
torch.cuda.synchronize()
e0.record()
for _ in range(10): m.tcl_topk_score(*args, ml, ks, res)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
out["topk_score_2000_tasks"] = {"ms": ms, "candidates": int(off[-1]), "Gcand_per_s": off[-1] / ms / 1e6}
print("topk_score", int(off[-1]), f"{ms:.3f} ms", flush=True)
json.dump(out, open("gpurun_out/next_rows_time.json", "w"), indent=1)

# KB + AC two-column inference vs the one-column model (fp32 path): paper and tuning configs
from paper_2604_12891_b200 import Model as _M
for name, n in (("paper", 16384), ("tuning", 16384)):
    c = inputs.config(name); d = c["dims"]; a = inputs.default_adapter_rank(d)
    kbw = inputs.make_weights(d, 1); acw = inputs.make_weights(d, 2); adw = inputs.make_adapters(d, a, 3)
    f, l = inputs.make_features(d, n, 5, workload="tuning")
    ft, lt = torch.from_numpy(f).cuda(), torch.from_numpy(l).cuda()
    s = torch.empty(n, device="cuda")
    for label, mm in (("one_column", _M(acw, d)), ("kb_ac", _M.kbac(kbw, acw, adw, a, d))):
        for _ in range(3): mm.tcl_score(ft, lt, s)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(10): mm.tcl_score(ft, lt, s)
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 10
        out[f"{name}_{label}"] = {"n": n, "ms": ms, "cand_per_s": n / ms * 1e3}
        print(name, label, f"{ms:.3f} ms", f"{n / ms * 1e3:.0f} cand/s", flush=True)
json.dump(out, open("gpurun_out/next_rows_time.json", "w"), indent=1)

# Training step (LambdaRank + backward + Adam), paper batch size 1024 in groups of 64
for name in ("paper", "tuning"):
    c = inputs.config(name); d = c["dims"]
    mm = _M(inputs.make_weights(d, 1), d)
    n = 1024
    f, l = inputs.make_features(d, n, 5, workload="tuning")
    rng = np.random.default_rng(0)
    lat = np.exp(rng.normal(-6, 0.7, n)).astype(np.float32)
    off = np.arange(0, n + 1, 64, dtype=np.int64)
    ft, lt, latt, offt = (torch.from_numpy(a).cuda() for a in (f, l, lat, off))
    mm.tcl_train_init(n)
    loss = torch.zeros(1, device="cuda")
    for _ in range(3): mm.tcl_train_step(ft, lt, latt, offt, 64, True, loss)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(10): mm.tcl_train_step(ft, lt, latt, offt, 64, True, loss)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    launches0 = mm.launch_count()
    mm.tcl_train_step(ft, lt, latt, offt, 64, True, loss); torch.cuda.synchronize()
    out[f"train_{name}_b1024"] = {"ms_per_step": ms, "cand_per_s": n / ms * 1e3,
                                  "launches_per_step": mm.launch_count() - launches0, "loss": float(loss.item())}
    print("train", name, f"{ms:.3f} ms/step", f"{n / ms * 1e3:.0f} cand/s", flush=True)
json.dump(out, open("gpurun_out/next_rows_time.json", "w"), indent=1)
