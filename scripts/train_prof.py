import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, inputs
from paper_2604_12891_b200 import Model
c = inputs.config(sys.argv[1] if len(sys.argv) > 1 else "paper"); d = c["dims"]
m = Model(inputs.make_weights(d, 1), d)
n = 1024
f, l = inputs.make_features(d, n, 5, workload="tuning")
lat = np.exp(np.random.default_rng(0).normal(-6, 0.7, n)).astype(np.float32)
off = np.arange(0, n + 1, 64, dtype=np.int64)
ft, lt, latt, offt = (torch.from_numpy(a).cuda() for a in (f, l, lat, off))
m.tcl_train_init(n)
loss = torch.zeros(1, device="cuda")
for _ in range(3): m.tcl_train_step(ft, lt, latt, offt, 64, True, loss)
torch.cuda.synchronize()
