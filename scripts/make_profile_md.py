#!/usr/bin/env python
"""Assemble profiles/<name>.md from a gpu_official.sh run (gpurun_out/): bench lines, launch list,
per-kernel ncu summaries, and refresh profiles/<traffic>.json (DRAM bytes per launch).

    python scripts/make_profile_md.py round1_ncu round1_traffic
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")


def run(*args):
    return subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "ncu_summary.py")] + list(args),
                          capture_output=True, text=True).stdout


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "round1_ncu"
    tname = sys.argv[2] if len(sys.argv) > 2 else "round1_traffic"
    prefix = sys.argv[3] if len(sys.argv) > 3 else "official"
    rnd = name.split("_")[0].replace("round", "Round ")
    parts = [f"# {rnd} — ncu evidence (large config: 65,536 candidates, L=64, d_model 256, 4 layers, bf16 projections)\n",
             f"Source: `scripts/gpu_official{'_r2' if prefix == 'r2' else ''}.sh` on one B200 via gpurun. Full captures: `ncu --set full --clock-control none "
             "--import-source on -k regex:<kernel> -s 4 -c 1 python bench.py --steps 1 --warmup 3`; launch list: `ncu "
             "--metrics gpu__time_duration.sum --clock-control none` over `bench.py --steps 2 --warmup 3`. ncu times are "
             "serialised and cold-cache: compare shares, not absolutes; bench.py's CUDA-event stage times are the live "
             "numbers. (k_ex2 / k_tanh / k_ffma / k_ffma2 are bench.py's peak microbenchmarks, run outside the timed "
             "region; k_pack / k_pool_bf16 captures use -s 3.)\n", "## Bench line of the same build\n"]
    for f in (f"bench_{prefix}.json", f"bench_reference_{prefix}.json", "bench_reference.json"):
        p = os.path.join(OUT, f)
        if os.path.exists(p):
            parts.append("```json\n" + open(p).read().strip() + "\n```\n")
    parts.append("## Launch list (all kernels of 2 timed + 3 warm-up steps + setup)\n")
    parts.append(run("launches", os.path.join(OUT, f"launches_{prefix}.csv")))
    parts.append("## Per-kernel full captures\n")
    reps = sorted(f for f in os.listdir(OUT) if f.startswith(f"prof_{prefix}_") and f.endswith(".ncu-rep"))
    order = ["k_scan", "k_inconv", "k_xdt", "k_gemm_ln", "k_enc12", "k_gemm_tc", "k_gemm_tf32", "k_head",
             "k_gemm_simt", "k_topk_radix", "k_pool_bf16", "k_pack"]
    reps.sort(key=lambda f: next((i for i, k in enumerate(order) if k in f), 99))
    for f in reps:
        parts.append(run("report", os.path.join(OUT, f)))
    open(os.path.join(ROOT, "profiles", name + ".md"), "w").write("\n".join(parts))
    # traffic per launch of the dominant kernels
    traffic = {}
    for key, rep in (("scan", "k_scan"), ("in_proj", "k_inconv"), ("xdt", "k_xdt"), ("out_proj", "k_gemm_ln"),
                     ("encoder", "k_enc12")):
        p = os.path.join(OUT, f"prof_{prefix}_{rep}.ncu-rep")
        if not os.path.exists(p):
            continue
        csv = subprocess.run(["ncu", "-i", p, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        lines = [l for l in csv.splitlines() if l.startswith('"')]
        hdr = [h.strip('"') for h in lines[0].split('","')]
        units = [h.strip('"') for h in lines[1].split('","')]
        row = [h.strip('"') for h in lines[2].split('","')]
        mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}

        def val(m):
            # exact metric name, else the (section-prefixed) column that ends with it
            i = hdr.index(m) if m in hdr else next(k for k, h in enumerate(hdr) if h.endswith(m))
            v = row[i].replace(",", "")
            return None if v == "no data" else float(v) * mult.get(units[i], 1)   # None: ncu had no sample
        traffic[key] = {"kernel": row[hdr.index("Kernel Name")][:60], "dram_bytes_read": val("dram__bytes_read.sum"),
                        "dram_bytes_write": val("dram__bytes_write.sum"),
                        # tcgen05 / mma.sync activity: the realtime tensor-pipe counter (the plain
                        # sm__pipe_tensor_cycles_active mirrors the XU issue counter on this part)
                        "tensor_pipe_pct": val("sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed"),
                        "xu_pipe_pct": val("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active"),
                        "source": f"profiles/{name}.md (prof_{prefix}_{rep}.ncu-rep)"}
    if traffic:
        json.dump(traffic, open(os.path.join(ROOT, "profiles", tname + ".json"), "w"), indent=1)
    print("wrote", name, list(traffic))


if __name__ == "__main__":
    main()
