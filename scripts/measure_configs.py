#!/usr/bin/env python
"""Per-config accuracy table for BASELINE.md §4: max |score_gpu - score_oracle| on a sample of each
BASELINE.json configuration (and top-k agreement), run on the GPU box.

    python scripts/measure_configs.py [--sample 512]
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import inputs  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sample", type=int, default=512)
    ap.add_argument("--full-large", action="store_true", help="score all 65,536 `large` candidates with the oracle")
    args = ap.parse_args()
    import torch
    from oracle import oracle as O
    from paper_2604_12891_b200 import Model
    wl = {"tiny": "tuning", "tuning": "tuning", "rdu": "rdu", "large": "large", "long": "long", "paper": "tuning"}
    out = {}
    for name in ("tiny", "tuning", "rdu", "large", "long", "paper"):
        c = inputs.config(name)
        d = c["dims"]
        w = inputs.make_weights(d, c["seed"])
        n = min(c["n"], args.sample if name == "long" or (name == "large" and not args.full_large) else c["n"])
        f, l = inputs.make_features(d, n, c["seed"] + 1, workload=wl[name])
        m = Model(w, d)
        ft, lt = torch.from_numpy(f).cuda(), torch.from_numpy(l).cuda()
        res = {"n": n, "precision": "bf16" if d.precision else "fp32"}
        if c["mc_passes"]:
            nn = min(n, 256)
            mean = torch.empty(nn, device="cuda")
            var = torch.empty(nn, device="cuda")
            m.tcl_score_mc(ft[:nn], lt[:nn], c["mc_passes"], 1234, 0, mean, var)
            m.tcl_sync_error()
            rm, rv = O.score_mc(d, w, f[:nn], l[:nn], c["mc_passes"], 1234, 0)
            res["mc_mean_max_abs_err"] = float(np.abs(mean.cpu().numpy() - rm).max())
            res["mc_var_max_abs_err"] = float(np.abs(var.cpu().numpy() - rv).max())
        s = torch.empty(n, device="cuda")
        m.tcl_score(ft, lt, s)
        m.tcl_sync_error()
        got = s.cpu().numpy()
        ref = O.score(d, w, f, l)
        err = np.abs(got - ref)
        res["max_abs_err"] = float(err.max())
        res["max_rel_err_vs_max1"] = float((err / np.maximum(1.0, np.abs(ref))).max())
        res["score_std"] = float(ref.std())
        res["max_abs_err_over_std"] = float(err.max() / ref.std())
        rel = err / np.maximum(np.abs(ref), 1e-30)
        res["rel_err_median"] = float(np.median(rel))
        res["rel_err_p99"] = float(np.percentile(rel, 99))
        rg = np.argsort(np.argsort(got, kind="stable"), kind="stable")
        rr = np.argsort(np.argsort(ref, kind="stable"), kind="stable")
        res["spearman"] = float(np.corrcoef(rg, rr)[0, 1])
        k = c["topk"] or 16
        gi = np.argsort(-got, kind="stable")[:k]
        ri, _ = O.topk(ref, k)
        res["topk_overlap"] = f"{len(set(gi) & set(ri))}/{k}"
        out[name] = res
        print(name, json.dumps(res), flush=True)
    json.dump(out, open(os.path.join(ROOT, "gpurun_out", "accuracy.json"), "w"), indent=1)


if __name__ == "__main__":
    main()
