#!/usr/bin/env python
"""Summarise ncu output into small text files for profiles/ (run here, on the CPU box).

    python scripts/ncu_summary.py launches gpurun_out/launches.csv  > profiles/rNN_launches.txt
    python scripts/ncu_summary.py kernel   gpurun_out/prof.ncu-rep   > profiles/rNN_<kernel>.txt

`launches`: per-kernel launch count, total and mean device time, share of all launches
(cold-cache, serialised: compare shares, not absolutes).
`kernel`: the headline metrics of each profiled launch (SOL, issue, occupancy, DRAM bytes,
L2 reds) plus instruction counts grouped by source line.
"""
from __future__ import annotations

import collections
import csv
import io
import subprocess
import sys


def launches(path: str) -> None:
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    hdr = rows[0]
    ix = {h: i for i, h in enumerate(hdr)}
    agg = collections.defaultdict(lambda: [0, 0.0])
    scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6, "s": 1e6}
    for r in rows[1:]:
        if r[ix["Metric Name"]] != "gpu__time_duration.sum":
            continue
        v = float(r[ix["Metric Value"]].replace(",", "")) * scale[r[ix["Metric Unit"]]]
        a = agg[r[ix["Kernel Name"]].split("(")[0][:100]]
        a[0] += 1
        a[1] += v
    tot = sum(v for _, v in agg.values())
    print(f"# {path}: {sum(n for n, _ in agg.values())} launches, {tot / 1e3:.3f} ms total (ncu, serialised, cold cache)")
    print(f"{'launches':>8} {'total_us':>11} {'mean_us':>9} {'share':>6}  kernel")
    for k, (n, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{n:8d} {v:11.1f} {v / n:9.2f} {100 * v / tot:5.1f}%  {k}")


KEYS = ["Duration", "Elapsed Cycles", "SM Frequency", "Compute (SM) Throughput", "Memory Throughput",
        "DRAM Throughput", "L1/TEX Cache Throughput", "L2 Cache Throughput", "Executed Ipc Active",
        "Issue Slots Busy", "No Eligible", "Eligible Warps Per Scheduler", "Warp Cycles Per Issued Instruction",
        "Avg. Active Threads Per Warp", "Executed Instructions", "Registers Per Thread",
        "Theoretical Occupancy", "Achieved Occupancy", "Grid Size", "Block Size", "L2 Hit Rate",
        "Dynamic Shared Memory Per Block", "Static Shared Memory Per Block"]
RAW = ["dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sectors_op_red.sum", "lts__t_requests_op_red.sum",
       "smsp__inst_executed_op_global_red.sum", "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
       "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
       "smsp__inst_executed.sum"]


def _ncu(args):
    return subprocess.run(["ncu", *args], capture_output=True, text=True).stdout


def kernel(path: str) -> None:
    det = list(csv.reader(io.StringIO(_ncu(["-i", path, "--page", "details", "--csv"]))))
    hdr = det[0]
    ix = {h: i for i, h in enumerate(hdr)}
    by_id = collections.OrderedDict()
    for r in det[1:]:
        by_id.setdefault(r[ix["ID"]], []).append(r)
    raw = list(csv.reader(io.StringIO(_ncu(["-i", path, "--page", "raw", "--csv"]))))
    rhdr = raw[0]
    for lid, rows in by_id.items():
        print(f"## launch {lid}: {rows[0][ix['Kernel Name']][:110]}")
        for r in rows:
            if r[ix["Metric Name"]] in KEYS:
                print(f"  {r[ix['Metric Name']]:40s} {r[ix['Metric Value']]:>16s} {r[ix['Metric Unit']]}")
        li = 2 + list(by_id).index(lid)
        if li < len(raw):
            for k in RAW:
                if k in rhdr:
                    j = rhdr.index(k)
                    print(f"  {k:60s} {raw[li][j]:>16s} {raw[1][j]}")
    src = list(csv.reader(io.StringIO(_ncu(["-i", path, "--page", "source", "--csv", "--print-source", "cuda,sass"]))))
    cur, h, agg, stall, text = None, None, collections.Counter(), collections.Counter(), {}
    for r in src:
        if r and r[0] == "File Path":
            cur = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            h = r
            continue
        if not r or r[0] in ("", "Function Name") or not h:
            continue
        try:
            ie = int(r[h.index("Instructions Executed")])
            st = int(r[h.index("Warp Stall Sampling (All Samples)")])
        except (ValueError, IndexError):
            continue
        key = (cur, int(r[0]))
        agg[key] += ie
        stall[key] += st
        text[key] = r[1].strip()[:80]
    tot, ts = sum(agg.values()) or 1, sum(stall.values()) or 1
    print(f"## source lines by executed warp instructions (all profiled launches: {tot} inst, {ts} stall samples)")
    for key, v in agg.most_common(40):
        print(f"  {100 * v / tot:5.1f}% inst {100 * stall[key] / ts:5.1f}% stall  {key[0]}:{key[1]:<4d} {text[key]}")


if __name__ == "__main__":
    {"launches": launches, "kernel": kernel}[sys.argv[1]](sys.argv[2])
