#!/usr/bin/env python
"""Executed warp instructions and stall samples of the fused raster kernel by code region.

    python scripts/ncu_regions.py gpurun_out/prof.ncu-rep

Regions are line ranges of csrc/raster.cu found by their marker comments (so they follow the
source), plus internal.cuh's band filter and exp2 helpers; the rest is 'other'."""
import collections
import csv
import io
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
MARKERS = [  # (region, regex of the first line)
    ("transpose_reduce", r"^__device__ __forceinline__ float transpose_reduce"),
    ("overflow", r"^__device__ __noinline__ void overflow_reds"),
    ("other", r"^static_assert\(BATCH == 32"),
    ("setup", r"// ---- setup: region id tuple"),
    ("refill", r"// ---- refill the ring"),
    ("superbatch_head", r"// a super-batch: up to NSUB"),
    ("warp_band_test", r"// ---- per-warp mask of sub-batch"),
    ("pixel_loop", r"// ---- rasterise: e\[j\]"),
    ("counters+overflow", r"// \(uncounted: the reductions run"),
    ("transpose+smem_acc", r"// ---- per \(warp, slot group\) transpose"),
    ("barrier+flush", r"// B: the super-batch's sums are complete"),
    ("epilogue", r"cp_async_wait_all\(\);  // no copy may land"),
]


def regions_of_raster():
    lines = open(os.path.join(ROOT, "paper_2605_13600_b200", "csrc", "raster.cu")).read().splitlines()
    starts = []
    for name, rx in MARKERS:
        for i, ln in enumerate(lines, 1):
            if re.search(rx, ln):
                starts.append((i, name))
                break
    starts.sort()
    return starts


def region(file, line, starts):
    if file == "internal.cuh":
        txt = open(os.path.join(ROOT, "paper_2605_13600_b200", "csrc", "internal.cuh")).read().splitlines()
        # the enclosing function's name
        for i in range(line - 1, -1, -1):
            m = re.match(r"^__device__ __forceinline__ \w+ (\w+)\(", txt[i])
            if m:
                return "internal:" + m.group(1)
        return "internal"
    if file != "raster.cu":
        return file
    name = "other"
    for s, n in starts:
        if line >= s:
            name = n
    return name


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    starts = regions_of_raster()
    agg, stall = collections.Counter(), collections.Counter()
    cur, h = None, None
    for r in csv.reader(io.StringIO(out)):
        if r and r[0] == "File Path":
            cur = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            h = r
            continue
        if not r or not h or r[0] in ("", "Function Name"):
            continue
        try:
            ie = int(r[h.index("Instructions Executed")])
            st = int(r[h.index("Warp Stall Sampling (All Samples)")])
        except (ValueError, IndexError):
            continue
        k = region(cur, int(r[0]), starts)
        agg[k] += ie
        stall[k] += st
    tot, ts = sum(agg.values()) or 1, sum(stall.values()) or 1
    print(f"# {path}: {tot} warp instructions, {ts} stall samples")
    for k, v in agg.most_common():
        print(f"  {100 * v / tot:5.1f}% inst  {100 * stall[k] / ts:5.1f}% stall  {k}")


if __name__ == "__main__":
    main(sys.argv[1])
