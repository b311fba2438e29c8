#!/usr/bin/env python
"""Summarise ncu reports / launch lists into the markdown tables kept under profiles/.

    python scripts/ncu_summary.py report REP.ncu-rep [...]      # per-kernel metrics + stall mix
    python scripts/ncu_summary.py launches LAUNCHES.csv          # per-kernel device-time shares
"""
import collections
import csv
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM %"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe %"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU (MUFU) inst %"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "L1 %"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 %"),
    ("sm__warps_active.avg.per_cycle_active", "warps/SM"),
    ("launch__registers_per_thread", "regs/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
]


def ncu_csv(args):
    out = subprocess.run(["ncu"] + args, capture_output=True, text=True).stdout
    return list(csv.reader(out.splitlines()))


def report(path):
    rows = ncu_csv(["-i", path, "--page", "raw", "--csv"])
    hdr, units = rows[0], rows[1]
    ix = {h: i for i, h in enumerate(hdr)}
    print(f"### {path.split('/')[-1]}\n")
    print("| kernel | " + " | ".join(name for _, name in METRICS) + " |")
    print("|---" * (len(METRICS) + 1) + "|")
    for r in rows[2:]:
        cells = []
        for key, _ in METRICS:
            if key in ix:
                v, u = r[ix[key]], units[ix[key]]
                cells.append(f"{v} {u}".strip())
            else:
                cells.append("-")
        print(f"| {r[ix['Kernel Name']][:48]} | " + " | ".join(cells) + " |")
    # stall mix from the source page
    src = ncu_csv(["-i", path, "--page", "source", "--csv", "--print-source", "sass"])
    blocks, cur = [], None
    for r in src:
        if r and r[0] == "Kernel Name":
            cur = [r]
            blocks.append(cur)
        elif cur is not None:
            cur.append(r)
    for b in blocks:
        if len(b) < 3:
            continue
        h = b[1]
        hix = {k: i for i, k in enumerate(h)}
        stalls = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
        agg = collections.Counter()
        for r in b[2:]:
            for k in stalls:
                try:
                    agg[k] += int(r[hix[k]] or 0)
                except (ValueError, IndexError):
                    pass
        tot = sum(agg.values()) or 1
        mix = ", ".join(f"{k[6:]} {v / tot:.0%}" for k, v in agg.most_common(6))
        print(f"\nstall mix ({b[0][1][:40]}): {mix}")
    print()


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10 and r[0] != "ID"]
    agg = collections.defaultdict(lambda: [0.0, 0])
    for r in rows:
        name = r[4].split("(")[0].replace("void ", "")
        unit, val = r[13], float(r[14].replace(",", ""))
        ns = val * (1000.0 if unit == "usecond" else 1.0) if unit in ("nsecond", "usecond") else val
        agg[name][0] += ns
        agg[name][1] += 1
    tot = sum(v[0] for v in agg.values())
    print(f"### {path.split('/')[-1]} (serialised, cold-cache per-launch times)\n")
    print("| kernel | launches | total us | share |")
    print("|---|---|---|---|")
    for k, (ns, n) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
        print(f"| {k} | {n} | {ns / 1e3:.1f} | {ns / tot:.1%} |")
    print()


if __name__ == "__main__":
    mode = sys.argv[1]
    for p in sys.argv[2:]:
        report(p) if mode == "report" else launches(p)
