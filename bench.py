#!/usr/bin/env python
"""bench.py -- throughput of the B200 scorer of TCL's Mamba cost model (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config large] [--impl ours|reference]

A "step" is one pass of the whole hot path over one batch of synthetic
candidates already resident in HBM: tcl_score (pack, encoder, n_layer Mamba blocks, head) followed
by tcl_topk (1 GPU) or tcl_topk_global (N GPUs: local top-k + ncclAllGather + merge).  Weak scaling:
every rank scores its own `n` candidates (global ids rank*n + i) and all ranks hold the identical
global top-k.  value = all candidates scored by all ranks / max-over-ranks device time.

Default workload: the `large batch` config of BASELINE.json (4-layer d_model=256 d_state=16,
65,536 candidates per GPU, seq len 64, bf16 projections).  One JSON line is printed by rank 0.
`--impl reference` times the fp64 CPU oracle (the reference arm of this tier) on bounded samples.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import inputs  # noqa: E402

METRIC = "candidate programs scored/sec at 1/2/4/8 B200; % of HBM/tensor-pipe roofline"
WORKLOAD_TEXT = {
    "tiny": "tiny: 1-layer Mamba d_model=64 d_state=16, 256 candidate programs, seq len 25, fp32",
    "tuning": "tuning round: 2-layer d_model=128, 4,096 candidates of one ResNet-50 conv2d subgraph, seq len 25, top-k=64",
    "rdu": "RDU uncertainty: 2-layer d_model=128, 16,384 candidates x 10 MC-dropout passes (mean/var scores)",
    "large": "large batch: 4-layer d_model=256 d_state=16, 65,536 candidates, seq len 64, bf16 projections",
    "long": "long-range schedules: 4-layer d_model=256, 1,048,576 candidates, seq len 128, global top-k=1024",
    "paper": "paper model [1,8,1,4] d_model=128, 26x22 CPU features",
}
FEATURE_WORKLOAD = {"tiny": "tuning", "tuning": "tuning", "rdu": "rdu", "large": "large", "long": "long",
                    "paper": "tuning"}


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        j = json.load(open(p))
        return dict(hbm=j["hbm_gbs"], bf16=j["bf16_tflops"], bf16_sus=j.get("bf16_tflops_sustained"),
                    sm_max_mhz=j.get("sm_max_mhz", 1965.0), source="measured (MEASURED_PEAKS.json)")
    return dict(hbm=6650.0, bf16=1590.0, bf16_sus=1400.0, sm_max_mhz=1965.0,
                source="fallback (B200_PROFILING.md)")


# ------------------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.t.join(timeout=2)
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------------------------------- roofline
def stage_model(d, P: int, n: int):
    """Algorithmic work per stage per launch: bytes that must cross HBM at the
    operand precision the kernel uses, flops of the dense contractions, MUFU exps of the scan."""
    dm, di, N, R = d.d_model, d.d_inner, d.d_state, d.dt_rank
    e1, e2 = d.enc_dims[0], d.enc_dims[1]
    act = 2 if d.precision == inputs.PREC_BF16_PROJ else 4
    bf16 = d.precision == inputs.PREC_BF16_PROJ
    nl = d.n_layer
    if bf16:
        # out_proj + fused LN (gemm_tc_ln): read g (bf16) and H (fp32); write H and LN_{l+1}(H) (bf16);
        # the last layer writes only LN_f(H) (bf16, the head's input).  Average per layer.
        out_bytes = (nl * (P * di * 2 + P * dm * 4) + (nl - 1) * (P * dm * 4 + P * dm * 2) + P * dm * 2) / nl
        head_bytes = P * dm * 2 + n * 4             # pool reads LN_f(H) bf16
        enc_bytes = P * 32 * 2 + P * dm * 4 + P * dm * 2   # X in; H and LN_0(H) out
    else:
        out_bytes = P * di * act + 2 * P * dm * 4
        head_bytes = P * dm * 4 + n * 4
        enc_bytes = P * 32 * act + P * dm * 4
    return {
        # pack: read the real rows of the padded fp32 features, write packed rows (32 cols)
        "pack": dict(bytes=P * d.d_in * 4 + P * 32 * act + n * 4),
        "encoder": dict(flops=2 * P * (32 * e1 + e1 * e2 + e2 * dm), bytes=enc_bytes),
        "layernorm": dict(bytes=P * dm * 4 + P * dm * act),
        # bf16 path: in_proj + SiLU(z) + conv + SiLU (k_inconv): LN(H) (bf16) in; SiLU(z) (bf16) and u
        # (fp16) out.  fp32 path: the in_proj GEMM ([x | z] fp32 out)
        "in_proj": (dict(flops=2 * P * dm * 2 * di, bytes=P * dm * 2 + P * di * 2 + P * di * 2) if bf16 else
                    dict(flops=2 * P * dm * 2 * di, bytes=P * dm * act + P * 2 * di * act)),
        "conv": dict(bytes=P * di * act + P * di * 4),
        "x_proj": dict(flops=2 * P * di * (R + 2 * N), bytes=P * di * 4 + P * (R + 2 * N) * 4),
        "dt_proj": dict(flops=2 * P * R * di, bytes=P * R * 4 + P * di * 4),
        # scan: u, delta, z in; g out (fp32) + B, C per token; N exps per (t, d).  bf16 path (split
        # mixer): the packet (u, Delta fp16, B, C fp32) and SiLU(z) (bf16) in, g (bf16) out
        "scan": (dict(bytes=P * (4 * di + 8 * N) + P * di * 2 + P * di * 2, exps=P * di * N) if bf16 else
                 dict(bytes=P * di * (3 * 4 + act) + P * 2 * N * 4, exps=P * di * N)),
        # bf16 path x_proj + dt_proj + softplus (k_xdt): u (fp16) in; Delta (fp16), B, C (fp32) out
        "xdt": dict(bytes=P * di * 2 + P * (2 * di + 8 * N), flops=2 * P * di * (R + 2 * N) + 2 * P * R * di),
        "out_proj": dict(flops=2 * P * di * dm, bytes=out_bytes),
        "head": dict(bytes=head_bytes),
        "mixer": dict(bytes=P * 2 * di * act + P * di * act, exps=P * di * N),
        "topk": dict(bytes=n * 4),
    }


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="large", choices=list(inputs.CONFIGS))
    ap.add_argument("--n", type=int, default=0, help="candidates per GPU (default: the config's)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--cpu-sample", type=int, default=0)
    ap.add_argument("--precision", choices=["config", "fp32", "bf16"], default="config",
                    help="override the configuration's precision (fp32 path / bf16 projections)")
    ap.add_argument("--scan", choices=["auto", "sequential", "chunked"], default="auto",
                    help="fp32-path recurrence (TCL_OPT_SCAN): by dims, sequential, or chunked across L")
    ap.add_argument("--scaling", choices=["weak", "strong"], default="weak",
                    help="weak: n candidates per GPU (default); strong: the config's n split over the GPUs "
                         "(SURVEY §8(e): rank r scores the contiguous shard r, global top-k over all)")
    args = ap.parse_args()
    if args.warmup < 3:
        print("warning: --warmup < 3 violates the timing rules; using 3", file=sys.stderr)
        args.warmup = 3

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    cfg = inputs.config(args.config)
    if args.precision != "config":
        cfg = dict(cfg, dims=cfg["dims"].replace(
            precision=inputs.PREC_BF16_PROJ if args.precision == "bf16" else inputs.PREC_FP32))
    d = cfg["dims"]
    n = args.n or cfg["n"]
    if args.config == "long" and not args.n:
        n = cfg["n"] // max(world, 8) if world > 1 else 131072   # 1M over 8 GPUs; 1/8 of it per GPU
    k = cfg["topk"] or 64

    if args.impl == "reference":
        return run_reference(args, cfg, d, n, k, world, rank)
    return run_ours(args, cfg, d, n, k, world, rank, local_rank)


def run_reference(args, cfg, d, n, k, world, rank):
    """Reference arm of this tier: the fp64 CPU oracle as it stands, on host cores, rank 0 only."""
    if rank != 0:
        return 0
    from oracle import oracle as O
    O.build()
    w = inputs.make_weights(d, cfg["seed"])
    sample = args.cpu_sample or {"tiny": 256, "tuning": 512, "rdu": 64, "paper": 256}.get(args.config, 256)
    sample = min(sample, n)
    f, l = inputs.make_features(d, sample, cfg["seed"] + 1, workload=FEATURE_WORKLOAD[args.config])
    cores = O.default_threads()
    passes = cfg["mc_passes"]

    def step():
        if passes:
            O.score_mc(d, w, f, l, passes, 1234, 0, nthreads=cores)
        else:
            s = O.score(d, w, f, l, nthreads=cores)
            O.topk(s, min(k, sample))

    for _ in range(args.warmup):
        step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    dt = (time.perf_counter() - t0) / args.steps
    value = sample / dt
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "candidates/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": WORKLOAD_TEXT[args.config], "n_per_step": sample,
                       "max_len": d.max_len, "d_model": d.d_model, "n_layer": d.n_layer,
                       "d_state": d.d_state, "mc_passes": passes},
            "cpu_baseline": {"value": value, "unit": "candidates/s", "cores": cores, "kind": "oracle",
                             "sample": f"{sample} candidates of the {args.config} workload per step "
                                       f"(fp64 C oracle, {cores} threads)", "cpu_model": cpu_model(),
                             "nproc": os.cpu_count()},
            "e2e": {"value": value, "unit": "candidates/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "gpu_launches": 0}
    print(json.dumps(line), flush=True)
    return 0


def run_ours(args, cfg, d, n, k, world, rank, local_rank):
    import torch
    import torch.distributed as dist
    from paper_2604_12891_b200 import Model, tcl_comm_unique_id

    torch.cuda.set_device(local_rank)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    peaks = load_peaks()
    w = inputs.make_weights(d, cfg["seed"])
    if args.scaling == "strong":
        # one global batch of n candidates, rank r takes its contiguous shard (global index = start + i)
        from paper_2604_12891_b200.tcl import shard_range
        fg, lg = inputs.make_features(d, n, cfg["seed"] + 1, workload=FEATURE_WORKLOAD[args.config])
        index_base, n_loc = shard_range(n, world, rank)
        feats, lens = np.ascontiguousarray(fg[index_base:index_base + n_loc]), lg[index_base:index_base + n_loc].copy()
        n_total = n
        n = n_loc
    else:
        feats, lens = inputs.make_features(d, n, cfg["seed"] + 1 + 7919 * rank, workload=FEATURE_WORKLOAD[args.config])
        index_base = rank * n
        n_total = n * world
    P = int(lens.sum())
    m = Model(w, d, device=local_rank)
    if args.scan != "auto":
        m.scan_mode(args.scan)
    m.reserve(n)
    if world > 1:
        obj = [tcl_comm_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        m.tcl_comm_init(obj[0], world, rank)

    stream = torch.cuda.Stream()
    feats_d = torch.from_numpy(feats).cuda()
    lens_d = torch.from_numpy(lens).cuda()
    scores_d = torch.empty(n, dtype=torch.float32, device="cuda")
    idx_d = torch.empty(k, dtype=torch.int64, device="cuda")
    top_d = torch.empty(k, dtype=torch.float32, device="cuda")
    mc = cfg["mc_passes"]
    var_d = torch.empty(n, dtype=torch.float32, device="cuda") if mc else None

    def step():
        if mc:
            m.tcl_score_mc(feats_d, lens_d, mc, 1234, index_base, scores_d, var_d, stream=stream)
        else:
            m.tcl_score(feats_d, lens_d, scores_d, stream=stream)
        if world > 1:
            m.tcl_topk_global(scores_d, index_base, k, idx_d, top_d, stream=stream)
        else:
            m.tcl_topk(scores_d, k, index_base, idx_d, top_d, stream=stream)

    torch.cuda.synchronize()
    for _ in range(args.warmup):
        step()
    m.tcl_sync_error(stream=stream)

    # ---------------- timed region (device time, CUDA events on the launching stream).  Repeated
    # calls replay CUDA graphs (TCL_OPT_GRAPHS, captured during the warm-up); every step recomputes
    # the whole path from the device-resident inputs.
    clocks = ClockSampler(local_rank)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.start()
    time.sleep(0.3)
    launches0 = m.launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for _ in range(args.steps):
        step()
    ev1.record(stream)
    torch.cuda.synchronize()
    launches = m.launch_count() - launches0
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    ms = ev0.elapsed_time(ev1)
    # ---------------- per-kernel device times: the same steps again with every launch bracketed by
    # CUDA events on the launching stream (direct launches; the headline number above is unprofiled)
    m.profile_enable(True)
    m.profile_read(reset=True)
    for _ in range(args.steps):
        step()
    torch.cuda.synchronize()
    prof = m.profile_read(reset=True)
    m.profile_enable(False)
    ms_prof = sum(v[0] for v in prof.values())
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_step = ms / args.steps
    value = n_total / (ms_step * 1e-3)

    # ---------------- roofline of the dominant kernel (live CUDA-event stage times)
    work = stage_model(d, P, n)
    mb = measured_issue_peaks()
    kernels = {}
    for kind, (tot_ms, cnt) in prof.items():
        per = tot_ms / cnt
        kernels[kind] = {"ms_per_launch": per, "launches": cnt, "share": tot_ms / ms_prof}
    per_step_launches = {kind: cnt / args.steps for kind, (_, cnt) in prof.items()}
    for kind, entry in kernels.items():
        wk = work.get(kind, {})
        calls = per_step_launches[kind]                  # launches of this stage per step
        units = (mc or 1) * (d.n_layer if kind in ("layernorm", "in_proj", "conv", "x_proj", "dt_proj",
                                                     "scan", "out_proj", "mixer", "xdt") else 1)
        scale = units / calls                            # fraction of a step's work per launch
        if "bytes" in wk:
            entry["gbs"] = wk["bytes"] * scale / (entry["ms_per_launch"] * 1e-3) / 1e9
            entry["hbm_frac"] = entry["gbs"] / peaks["hbm"]
        if "flops" in wk:
            entry["tflops"] = wk["flops"] * scale / (entry["ms_per_launch"] * 1e-3) / 1e12
        if "exps" in wk:
            entry["ex2_per_s"] = wk["exps"] * scale / (entry["ms_per_launch"] * 1e-3)
            entry["sfu_frac"] = entry["ex2_per_s"] / mb["ex2"]
            if mb.get("scanmix"):
                entry["scanmix_frac"] = entry["ex2_per_s"] / mb["scanmix"]
    dom = max(kernels, key=lambda kk: kernels[kk]["share"])
    de = kernels[dom]
    wk = work[dom]
    calls = per_step_launches[dom]
    units = (mc or 1) * (d.n_layer if dom in ("layernorm", "in_proj", "conv", "x_proj", "dt_proj", "scan",
                                                "out_proj", "mixer", "xdt") else 1)
    traffic = None  # DRAM bytes per launch of this kernel from one ncu --set full capture (profiles/)
    tp = os.path.join(ROOT, "profiles", "round2_traffic.json")
    if not os.path.exists(tp):
        tp = os.path.join(ROOT, "profiles", "round1_traffic.json")
    if os.path.exists(tp):
        tall = json.load(open(tp))
        tj = tall.get(dom)
        if tj and args.config == "large":
            traffic = tj["dram_bytes_read"] + tj["dram_bytes_write"]
        # per-stage pipe utilisation of the same ncu captures (tensor pipe of the projections, XU of the
        # scan): ncu-sourced, at this configuration only
        if args.config == "large" and d.precision == inputs.PREC_BF16_PROJ:
            for kind, entry in kernels.items():
                tk = tall.get(kind)
                if tk and "tensor_pipe_pct" in tk:
                    entry["ncu"] = {"tensor_pipe_pct": tk["tensor_pipe_pct"], "xu_pipe_pct": tk.get("xu_pipe_pct"),
                                    "dram_bytes_per_launch": tk["dram_bytes_read"] + tk["dram_bytes_write"],
                                    "source": tk.get("source")}
    if "exps" in wk:
        roof = {"bound": "alu", "achieved": de["ex2_per_s"] / 1e12, "peak": mb["ex2"] / 1e12,
                "unit": "Tex2/s", "frac": de["sfu_frac"],
                "traffic": traffic, "kernel": dom,
                "peak_source": mb["source"],
                "algorithmic_units_per_launch": wk["exps"] * units / calls,
                # the scan's own instruction mix (2 MUFU.EX2 + 6 packed FMA-pipe ops per state pair,
                # microbench k_scanmix at the mixer's 16 warps/SM) cannot reach the MUFU-only peak
                "scan_mix": ({"peak": mb["scanmix"] / 1e12, "frac": de["ex2_per_s"] / mb["scanmix"],
                              "unit": "Tex2/s", "source": "measured (microbench k_scanmix)"}
                             if mb.get("scanmix") else None),
                "hbm": {"achieved_gbs": de.get("gbs"), "peak_gbs": peaks["hbm"], "frac": de.get("hbm_frac"),
                        "algorithmic_bytes_per_launch": wk["bytes"] * units / calls}}
    elif "flops" in wk and d.precision == inputs.PREC_BF16_PROJ and dom in ("in_proj", "out_proj", "encoder"):
        roof = {"bound": "tensor", "achieved": de["tflops"], "peak": peaks["bf16"], "unit": "TFLOP/s",
                "frac": de["tflops"] / peaks["bf16"], "traffic": None, "kernel": dom,
                "peak_source": peaks["source"]}
    elif "flops" in wk:
        roof = {"bound": "alu", "achieved": de["tflops"], "peak": mb["ffma"] * 2 / 1e12, "unit": "TFLOP/s",
                "frac": de["tflops"] / (mb["ffma"] * 2 / 1e12), "traffic": None, "kernel": dom,
                "peak_source": mb["source"] + " (FFMA lanes x 2)"}
    else:
        roof = {"bound": "hbm", "achieved": de["gbs"], "peak": peaks["hbm"], "unit": "GB/s",
                "frac": de["gbs"] / peaks["hbm"], "traffic": None, "kernel": dom, "peak_source": peaks["source"]}

    # ---------------- end-to-end through the host API (pinned host buffers, H2D + D2H timed)
    e2e = None
    if not args.no_e2e:
        fp = torch.from_numpy(feats).pin_memory()
        lp = torch.from_numpy(lens).pin_memory()
        sp = torch.empty(n, dtype=torch.float32).pin_memory()
        ip = torch.empty(k, dtype=torch.int64).pin_memory()
        tp = torch.empty(k, dtype=torch.float32).pin_memory()
        fnp, lnp, snp, inp, tnp = fp.numpy(), lp.numpy(), sp.numpy(), ip.numpy(), tp.numpy()
        vp = torch.empty(n, dtype=torch.float32).pin_memory() if mc else None

        def e2e_step():
            if not mc:   # the host-buffer call: pipelined H2D, scoring, top-k, D2H
                m.tcl_score_host(fnp, lnp, k, index_base, snp, inp, tnp, stream=stream)
                return
            # MC (no host-buffer variant): H2D of the step's inputs, tcl_score_mc, top-k of the means,
            # D2H of mean / var / top-k, all on the scoring stream
            with torch.cuda.stream(stream):
                feats_d.copy_(fp, non_blocking=True)
                lens_d.copy_(lp, non_blocking=True)
            m.tcl_score_mc(feats_d, lens_d, mc, 1234, index_base, scores_d, var_d, stream=stream)
            m.tcl_topk(scores_d, k, index_base, idx_d, top_d, stream=stream)
            with torch.cuda.stream(stream):
                sp.copy_(scores_d, non_blocking=True)
                vp.copy_(var_d, non_blocking=True)
                ip.copy_(idx_d, non_blocking=True)
                tp.copy_(top_d, non_blocking=True)
            stream.synchronize()

        for _ in range(args.warmup):
            e2e_step()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            e2e_step()
        e1.record(stream)
        torch.cuda.synchronize()
        ems = e0.elapsed_time(e1)
        if world > 1:
            t = torch.tensor([ems], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ems = float(t.item())
        e2e = {"value": n_total / (ems / args.steps * 1e-3), "unit": "candidates/s",
               "h2d_bytes_per_step": int(feats.nbytes + lens.nbytes),
               "d2h_bytes_per_step": int(n * 4 * (2 if mc else 1) + k * 12),
               "ms_per_step": ems / args.steps}

    # ---------------- CPU baseline: the oracle on host cores, rank 0 at N=1 only
    cpu = None
    if world == 1 and rank == 0 and not args.no_cpu_baseline:
        from oracle import oracle as O
        O.build()
        # bounded sample: ~10-20 s of CPU work on the GPU box's host cores
        sample = args.cpu_sample or {"tiny": 256, "tuning": 4096, "rdu": 512, "large": 6144,
                                     "long": 1536, "paper": 4096}[args.config]
        sample = min(sample, n)
        cores = O.default_threads()
        t0 = time.perf_counter()
        if mc:
            O.score_mc(d, w, feats[:sample], lens[:sample], mc, 1234, 0, nthreads=cores)
        else:
            O.score(d, w, feats[:sample], lens[:sample], nthreads=cores)
        dt = time.perf_counter() - t0
        # one thread on a sixteenth of the sample (the per-core rate)
        s1 = max(1, sample // 16)
        t1 = time.perf_counter()
        if mc:
            O.score_mc(d, w, feats[:s1], lens[:s1], mc, 1234, 0, nthreads=1)
        else:
            O.score(d, w, feats[:s1], lens[:s1], nthreads=1)
        dt1 = time.perf_counter() - t1
        cpu = {"value": sample / dt, "unit": "candidates/s", "cores": cores, "kind": "oracle",
               "sample": f"first {sample} of the {n} candidates of this workload "
                         f"(fp64 C oracle, gcc -O2, {cores} threads, {dt:.1f} s)",
               "cpu_model": cpu_model(), "nproc": os.cpu_count(),
               "one_thread": {"value": s1 / dt1, "unit": "candidates/s", "sample": f"first {s1} candidates, 1 thread, {dt1:.1f} s"}}

    if rank == 0:
        dtype = "bf16+f32" if d.precision == inputs.PREC_BF16_PROJ else "f32"
        line = {
            "metric": METRIC, "value": value, "unit": "candidates/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None,
            "dtype": dtype, "data": "synthetic",
            "config": {"workload": WORKLOAD_TEXT[args.config], "config": args.config,
                       "precision": "bf16 projections" if d.precision == inputs.PREC_BF16_PROJ else "fp32",
                       "n_per_gpu": n, "global_n": n_total, "packed_tokens_per_gpu": P,
                       "max_len": d.max_len, "d_model": d.d_model, "n_layer": d.n_layer,
                       "d_state": d.d_state, "topk": k, "mc_passes": mc,
                       "parallelism": f"dp{world} (candidate shards, all-gather top-k)",
                       "l2": f"inputs larger than L2: {feats.nbytes / 1e6:.0f} MB features per GPU per step"},
            "roofline": roof,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches,
            "clocks": clk,
            "kernels": kernels,
            "kernel_times": "per-launch CUDA events on the launching stream, in a re-run of the timed steps "
                            "with direct launches (the timed steps replay CUDA graphs)",
            "peaks": {"hbm_gbs": peaks["hbm"], "bf16_tflops": peaks["bf16"], "ex2_per_s": mb["ex2"],
                      "ffma_per_s": mb["ffma"], "ffma2_lanes_per_s": mb.get("ffma2"),
                      "tanh_per_s": mb.get("tanh"), "scanmix_ex2_per_s": mb.get("scanmix"), "source": peaks["source"], "issue_source": mb["source"]},
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


_MB = None


def measured_issue_peaks():
    """MUFU.EX2 and FFMA chip throughput measured on this GPU (libtcl_microbench.so)."""
    global _MB
    if _MB is not None:
        return _MB
    import ctypes
    derived = {"ex2": 148 * 16 * 1.965e9, "ffma": 148 * 128 * 1.965e9,
               "source": "derived: 148 SM x 16 ex2/clk (x 128 FFMA/clk) x 1965 MHz"}
    p = os.path.join(ROOT, "paper_2604_12891_b200", "libtcl_microbench.so")
    try:
        L = ctypes.CDLL(p)
        L.tclmb_run.restype = ctypes.c_double
        L.tclmb_run.argtypes = [ctypes.c_int, ctypes.c_int]
        ex2 = L.tclmb_run(0, 4096)
        ffma = L.tclmb_run(1, 8192)
        ffma2 = L.tclmb_run(2, 8192)
        tanh = L.tclmb_run(3, 4096)
        scanmix = L.tclmb_run(4, 2048)
        if ex2 > 0 and ffma > 0:
            _MB = {"ex2": ex2, "ffma": ffma, "ffma2": ffma2, "tanh": tanh, "scanmix": scanmix if scanmix > 0 else None,
                   "source": "measured (microbench: 148x8 CTAs x 256 thr, 8 chains)"}
            return _MB
    except OSError:
        pass
    _MB = derived
    return _MB


if __name__ == "__main__":
    sys.exit(main())
