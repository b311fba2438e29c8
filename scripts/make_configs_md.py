#!/usr/bin/env python
"""Assemble profiles/round1_configs.md from a gpu_official.sh run (gpurun_out/bench_*.json).

    python scripts/make_configs_md.py [name]
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")


def row(name, prec, d):
    r = d["roofline"]
    st = ", ".join(f"{k} {v['ms_per_launch']:.3f}" for k, v in d["kernels"].items())
    return (f"| {name} | {prec} | {d['value']:,.0f} | {d['ms_per_step']:.3f} | {d['e2e']['value']:,.0f} | "
            f"{r['kernel']} | {r['frac']:.3f} of {r['peak']:.4g} {r['unit']} ({r['bound']}) | {st} |")


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "round1_configs"
    out = ["# Round 1 — every BASELINE.json configuration on one B200 (`bench.py --config C --precision P`)\n",
           "Source: `scripts/gpu_official.sh` (same build as `round1_ncu.md`). 20 timed steps after 3 warm-ups "
           "(long: 5), CUDA events, inputs resident in HBM (`value`); `e2e` = the host API with pinned host buffers, "
           "H2D + D2H inside the timed region (host-latency-bound for the small configurations). `fp32` = the 1e-4 "
           "parity path (CUDA-core GEMMs); `bf16` = bf16 projections on tcgen05 (2e-2 parity path). Stage times are "
           "per launch.\n",
           "| config | precision | candidates/s | ms / step | e2e candidates/s | dominant kernel | its roofline fraction | stage ms / launch |",
           "|---|---|---|---|---|---|---|---|"]
    for c in ("tiny", "tuning", "rdu", "paper"):
        for pr in ("fp32", "bf16"):
            p = os.path.join(OUT, f"bench_{c}_{pr}.json")
            if os.path.exists(p):
                d = json.load(open(p))
                mc = d["config"].get("mc_passes", 0)
                out.append(row(c + (f" ({mc} MC passes)" if mc else ""), pr, d))
    for label, f in (("large (bench default)", "bench_official.json"), ("long, 131,072 per GPU", "bench_long.json")):
        p = os.path.join(OUT, f)
        if os.path.exists(p):
            out.append(row(label, "bf16", json.load(open(p))))
    out.append("\nAccuracy against the fp64 oracle (`scripts/measure_configs.py`, same run): "
               "`profiles/round1_accuracy.json`, summarised in BASELINE.md §4.\n")
    open(os.path.join(ROOT, "profiles", name + ".md"), "w").write("\n".join(out) + "\n")
    print("\n".join(out[4:]))


if __name__ == "__main__":
    main()
