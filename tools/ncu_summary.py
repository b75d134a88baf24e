#!/usr/bin/env python3
"""Summarise ncu captures into the markdown kept under profiles/.

    python tools/ncu_summary.py launches <launches.csv>           # per-launch times and shares
    python tools/ncu_summary.py kernel <report.ncu-rep> [flops]   # key metrics + stall breakdown

Reads reports with `ncu -i ... --page raw/source --csv` (no GPU needed).
"""
import csv
import io
import subprocess
import sys
from collections import Counter, defaultdict

KEYS = [
    "gpu__time_duration.sum",
    "sm__cycles_elapsed.avg.per_second",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_sector_hit_rate.pct",
    "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__ops_path_tensor_src_fp64.sum",
    "sm__ops_path_tensor_src_fp64.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active",
    "lts__t_bytes.sum",
    "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
    "smsp__inst_executed.sum",
    "sm__issue_active.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "launch__registers_per_thread",
    "launch__grid_size",
    "launch__block_size",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
]


def ncu_csv(rep, page, extra=()):
    out = subprocess.run(["ncu", "-i", rep, "--page", page, "--csv", *extra],
                         capture_output=True, text=True, check=True).stdout
    return list(csv.reader(io.StringIO(out)))


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    per = defaultdict(list)
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d["Metric Name"] != "gpu__time_duration.sum":
                continue
            name = d["Kernel Name"].split("(")[0].replace("void ", "")
            per[name].append(float(d["Metric Value"]) * (1e-3 if d["Metric Unit"] == "ns" else
                                                         1.0 if d["Metric Unit"] == "us" else 1e3))
    tot = sum(sum(v) for v in per.values())
    print("| kernel | launches | mean us | total ms | share |")
    print("|---|---|---|---|---|")
    for k, v in sorted(per.items(), key=lambda kv: -sum(kv[1])):
        print(f"| `{k}` | {len(v)} | {sum(v)/len(v):.1f} | {sum(v)/1e3:.3f} | {100*sum(v)/tot:.2f} % |")


def kernel(rep, flops=None):
    rows = ncu_csv(rep, "raw")
    hdr, units, vals = rows[0], rows[1], rows[2]
    name = vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
    print(f"kernel: `{name[:120]}`\n")
    print("| metric | value | unit |")
    print("|---|---|---|")
    got = {}
    for h, u, v in zip(hdr, units, vals):
        if h in KEYS:
            got[h] = (v, u)
    for k in KEYS:
        if k in got:
            print(f"| {k} | {got[k][0]} | {got[k][1]} |")
    if flops and "gpu__time_duration.sum" in got:
        v, u = got["gpu__time_duration.sum"]
        t = float(v) * {"s": 1, "ms": 1e-3, "us": 1e-6, "ns": 1e-9}.get(u, 1)
        print(f"\nalgorithmic work {float(flops):.4g} flop / {t:.4f} s = {float(flops)/t/1e12:.2f} TFLOP/s")
    src = ncu_csv(rep, "source", ["--print-source", "sass"])
    h = src[1]
    idx = {x: i for i, x in enumerate(h)}
    ops = Counter()
    tot = 0
    for r in src[2:]:
        if len(r) < len(h):
            continue
        try:
            smp = int(r[idx["Warp Stall Sampling (All Samples)"]] or 0)
        except ValueError:
            continue
        ins = r[idx["Source"]].strip()
        op = ins.split()[1] if ins.startswith("@") else (ins.split()[0] if ins else "?")
        ops[op.split(".")[0]] += smp
        tot += smp
    print("\nwarp-state samples by SASS opcode (top 12):\n")
    print("| opcode | share |")
    print("|---|---|")
    for op, c in ops.most_common(12):
        print(f"| {op} | {100*c/tot:.1f} % |")


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2])
    else:
        kernel(sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else None)
