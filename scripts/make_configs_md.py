#!/usr/bin/env python
"""Assemble profiles/<name>.md from a gpu_official_r2.sh run (gpurun_out/bench_*.json): every
BASELINE.json configuration's bench line.

    python scripts/make_configs_md.py round2_configs
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")


def row(name, prec, d):
    steps = d["steps"]
    tot = sum(v["ms_per_launch"] * v["launches"] for v in d["kernels"].values())
    top = sorted(d["kernels"].items(), key=lambda kv: -kv[1]["ms_per_launch"] * kv[1]["launches"])[:3]
    st = ", ".join(f"{k} {100 * v['ms_per_launch'] * v['launches'] / tot:.0f}%" for k, v in top)
    e2e = d.get("e2e") or {}
    e2e_v = f"{e2e['value'] / 1e6:.2f} M" if e2e.get("value") else "-"
    return (f"| {name} | {prec} | {d['value'] / 1e6:.2f} M | {d['ms_per_step']:.4g} | {e2e_v} | "
            f"{d['gpu_launches'] / steps:.0f} | {st} |")


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "round2_configs"
    rnd = name.split("_")[0].replace("round", "Round ")
    out = [f"# {rnd} — every configuration (one B200, `scripts/configs_gpu.sh` inside `scripts/gpu_official_r2.sh`)\n",
           "`python bench.py --config C --precision P --steps 20 --warmup 3`; timed region = CUDA-graph replays of the "
           "repeated calls (captured during warm-up); e2e = `tcl_score_host` with pinned host buffers, H2D + D2H inside "
           "the timed region.  Accuracy per config: `round2_accuracy.json`.\n",
           "| config | precision | candidates/s | ms / step | e2e candidates/s | launches / step | top stages (profiled re-run) |",
           "|---|---|---|---|---|---|---|"]
    for c in ("tiny", "tuning", "rdu", "paper"):
        for pr in ("fp32", "bf16"):
            p = os.path.join(OUT, f"bench_{c}_{pr}.json")
            if os.path.exists(p):
                out.append(row(c, pr, json.load(open(p))))
    for label, f in (("long (131,072 per GPU)", "bench_long.json"), ("**large**", "bench_r2.json")):
        p = os.path.join(OUT, f)
        if os.path.exists(p):
            out.append(row(label, "bf16", json.load(open(p))))
    open(os.path.join(ROOT, "profiles", name + ".md"), "w").write("\n".join(out) + "\n")
    print("\n".join(out[2:]))


if __name__ == "__main__":
    main()
