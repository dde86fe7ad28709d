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


MARKERS2 = [  # raster2.cu (the production kernel)
    ("transpose8", r"^__device__ __forceinline__ float transpose8"),
    ("pass_select", r"^__device__ __forceinline__ float pass_select"),
    ("overflow", r"^__device__ __noinline__ void overflow_red1"),
    ("setup", r"^__global__ void __launch_bounds__\(R2T"),
    ("refill", r"// ---- refill the ring"),
    ("superbatch_head", r"const uint32_t n = min\(\(uint32_t\)R2SB, q_count\);"),
    ("warp_band_test", r"const uint32_t sh = "),
    ("group_loop_head", r"for \(int g0 = 0; g0 < BATCH; g0 \+= RG\)"),
    ("pixel_loop", r"float eA\[RG\], eB\[RG\];"),
    ("reduce+smem_acc", r"// ---- reduce the group's weights"),
    ("barrier", r"// the super-batch's sums are complete"),
    ("flush", r"// ---- flush: S reds per"),
    ("flush_zero+advance", r"// zero the buffer of super-batch i\+2"),
    ("epilogue", r"cp_async_wait_all\(\);  // no copy may land"),
]


def regions_of_raster(fname="raster.cu", markers=None, text=None):
    markers = markers or MARKERS
    lines = (text or open(os.path.join(ROOT, "paper_2605_13600_b200", "csrc", fname)).read()).splitlines()
    starts = []
    for name, rx in markers:
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
    if file == "raster2.cu" and STARTS2:
        name = "other"
        for s, n in STARTS2:
            if line >= s:
                name = n
        return "r2:" + name
    if file != "raster.cu":
        return file
    name = "other"
    for s, n in starts:
        if line >= s:
            name = n
    return name


STARTS2 = []


def main(path, rev=None):
    global STARTS2
    # raster2.cu as profiled: the working tree, or `rev` (a git revision) when the capture is older
    text = None
    if rev:
        text = subprocess.run(["git", "-C", ROOT, "show", f"{rev}:paper_2605_13600_b200/csrc/raster2.cu"],
                              capture_output=True, text=True).stdout
    STARTS2 = regions_of_raster("raster2.cu", MARKERS2, text)
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
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else None)
