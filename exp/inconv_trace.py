"""Phase timeline of k_inconv (experiment): run the `large` bf16 forward through exp/libtcl_trace.so and
print per-phase cycle deltas (median over the first tiles of CTAs 0 and 1)."""
import ctypes, os, sys
import numpy as np
HERE = os.path.dirname(os.path.abspath(__file__))
os.environ["TCL_LIB"] = os.path.join(HERE, "libtcl_trace.so")
sys.path.insert(0, os.path.dirname(HERE))
import torch
import inputs
from paper_2604_12891_b200 import Model, tcl

name = sys.argv[1] if len(sys.argv) > 1 else "large"
c = inputs.config(name)
d = c["dims"].replace(precision=inputs.PREC_BF16_PROJ)
w = inputs.make_weights(d, c["seed"])
n = c["n"] if "n" in c else 65536
f, l = inputs.make_features(d, n, c["seed"] + 1, workload=name)
m = Model(w, d)
ft, lt = torch.from_numpy(f).cuda(), torch.from_numpy(l).cuda()
s = torch.empty(n, dtype=torch.float32, device="cuda")
for _ in range(3):
    m.tcl_score(ft, lt, s)
torch.cuda.synchronize()
L = tcl.load()
buf = np.zeros((2, 256, 8), dtype=np.uint64)
assert L.tcl_diag_inconv_trace(ctypes.c_void_p(buf.ctypes.data)) == 0
names = {0: "iter", 1: "afull", 2: "stg free", 3: "x staged", 6: "x loaded", 4: "conv done", 5: "end"}
for cta in range(2):
    t = buf[cta].astype(np.int64)
    ok = t[:, 0] > 0
    t = t[ok]
    print(f"CTA {cta}: {len(t)} tiles; per-tile period (cycles): {np.median(np.diff(t[:, 0])):.0f}")
    seq = [0, 1, 2, 3, 6, 4, 5]
    for a, b in zip(seq, seq[1:]):
        dd = t[1:, b] - t[1:, a]
        print(f"  {names[a]:>12} -> {names[b]:<12} median {np.median(dd):8.0f}  p90 {np.percentile(dd, 90):8.0f}")
    print("  mma(j) start - iter(j) start:", np.median(t[1:, 7] - t[1:, 0]))
