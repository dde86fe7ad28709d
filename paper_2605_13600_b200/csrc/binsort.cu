// binsort.cu -- per-bin depth-ordered Gaussian lists of a depth chunk by a stable counting sort
// (DESIGN.md §5 a3).  This is the binning step the paper inherits from the 3DGS rasteriser
// (Gaussians "sorted ... per tile by depth"); here the chunk's selected elements
// are already in (view, depth, index) order (one radix sort of their depth keys), and every
// element covers a rectangle of bins, so each bin's list is the subsequence of that order
// covering the bin.  Instead of expanding (bin, element) entries and radix-sorting them by bin,
// the lists are written straight to their final positions.  The chunk's entries, flattened in
// element order (an element's bins row-major over its rectangle), are cut per view into
// segments of BS_SEGE entries or more (equal work: the nearest Gaussians cover many bins):
//
//   bs_gather   entry counts in sorted order (-> CUB inclusive scan: offs) and their u64 total;
//   bs_views    per view: sorted-element range (from the compaction's view offsets), entry range
//               and first segment;
//   bs_count    one warp per segment: its first element (binary search of offs), then its
//               entries in order, 32 per step (owner element by a warp search of the prefixes):
//               the flattened (bin, element) pairs (coalesced, 6 B) and per-bin entry counts of
//               the segment (a shared-memory row of the view's bins) -> the [segment][bin]
//               count matrix;
//   bs_colscan  per (view, bin): exclusive scan of the counts over the view's segments (in place;
//               8 warps per 32 bins, each a contiguous part of the segments) and the bin's total;
//   bs_ranges   per view: exclusive scan of the bin totals + the view's entry base -> ranges;
//   bs_scatter  one warp per segment again, reading its flattened entries IN ORDER with a row of
//               running positions (range start + column prefix): every 32 consecutive entries
//               are ranked within their bin by warp match (earlier lanes = earlier elements, and
//               an element covers a bin once), so each list keeps the sorted order (stable).
//
// Traffic per entry: 6 B written + read (flattened pairs), 4 B written (the bin lists); per
// element 4 + 4 + 8 B read (offset, order, rectangle); per segment 3 x 4 B per bin of its view
// (count matrix write, scan, read).
#include <cub/block/block_scan.cuh>

#include <algorithm>

#include "internal.cuh"

namespace scoup {

namespace {

constexpr unsigned FULL = 0xffffffffu;
constexpr int BS_WARPS_MAX = 8;
// a view has at most MAX_SAT_ENTRIES 16x16 tiles and bins are >= 1 tile: one warp's row fits
static_assert(MAX_SAT_ENTRIES * 5 <= 200 * 1024, "bin row (+ lane tags) in shared memory");

// The segment of warp `seg`: its view and entry range [q0, q1) (chunk-flattened positions).
__device__ __forceinline__ bool bs_segment(const BsInfo* info, int nv, uint32_t seg, int& v, uint32_t& q0,
                                           uint32_t& q1) {
    if (seg >= info->segbase[nv]) return false;
    v = 0;
    for (int u = 1; u < nv; u++)
        if (info->segbase[u] <= seg) v = u;  // the last view starting at or before seg (empty views skipped)
    q0 = info->ebase[v] + (seg - info->segbase[v]) * info->sege;
    q1 = min(q0 + info->sege, info->ebase[v + 1]);
    return true;
}

// First sorted element of view v whose entries reach past q (offs: inclusive entry prefix).
__device__ __forceinline__ uint32_t bs_first_element(const uint32_t* __restrict__ offs, const BsInfo* info, int v,
                                                     uint32_t q) {
    uint32_t lo = info->vstart[v], hi = info->vstart[v + 1];
    while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (__ldg(offs + mid) <= q) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

// Walk entries [q0, q1) of view v in order, 32 per step, starting at sorted element k (the one
// holding q0): f(valid, bin within the view, element index).
template <class F>
__device__ __forceinline__ void bs_walk(uint32_t k, uint32_t kend, uint32_t q0, uint32_t q1,
                                        const uint32_t* __restrict__ offs, const uint32_t* __restrict__ sval_sorted,
                                        const uint2* __restrict__ rect, int bins_x, F&& f) {
    const int lane = threadIdx.x & 31;
    // group of 32 elements from k: inclusive / exclusive entry prefixes, index, rectangle; the next
    // group's prefixes and indices are loaded while this one is walked (latency of the chains)
    auto load = [&](uint32_t kb, uint32_t& inc, uint32_t& exc, uint32_t& e) {
        const uint32_t kk = kb + (uint32_t)lane;
        inc = 0xFFFFFFFFu;
        e = 0;
        if (kk < kend) {
            inc = __ldg(offs + kk);
            e = __ldg(sval_sorted + kk);
        }
        exc = (kk > 0 && kk <= kend) ? __ldg(offs + kk - 1) : 0u;
    };
    uint32_t inc, exc, e;
    load(k, inc, exc, e);
    uint32_t q = q0;
    while (q < q1) {
        uint2 rc = make_uint2(0u, 1u);
        if (inc > exc && inc != 0xFFFFFFFFu) rc = __ldg(rect + e);
        // m / w by multiply-high with ceil(2^32 / w), once per element (exact: m, w <= 12288)
        const uint32_t wl = (rc.y & 0xFFFFu) - (rc.x & 0xFFFFu);
        const uint32_t mg = wl > 1u ? 0xFFFFFFFFu / wl + 1u : 0u;
        uint32_t n_inc, n_exc, n_e;
        load(k + 32, n_inc, n_exc, n_e);
        const uint32_t last = __shfl_sync(FULL, inc, 31);  // entries of these 32 elements end here
        const uint32_t qe = min(q1, last);
        for (; q < qe; q += 32) {
            const uint32_t qq = q + (uint32_t)lane;
            // owner lane of entry qq: the number of lanes whose inclusive prefix is <= qq
            int l = 0;
#pragma unroll
            for (int step = 16; step; step >>= 1) {
                const uint32_t Pc = __shfl_sync(FULL, inc, l + step - 1);
                if (Pc <= qq) l += step;
            }
            const uint32_t ex = __shfl_sync(FULL, exc, l);
            const uint32_t rx = __shfl_sync(FULL, rc.x, l), ry = __shfl_sync(FULL, rc.y, l);
            const uint32_t el = __shfl_sync(FULL, e, l);
            const uint32_t ml = __shfl_sync(FULL, mg, l);
            const bool valid = qq < qe;
            uint32_t b = 0xFFFFFFFFu;
            if (valid) {
                const uint32_t m = qq - ex;
                const uint32_t bx0 = rx & 0xFFFFu, by0 = rx >> 16, w = (ry & 0xFFFFu) - bx0;
                const uint32_t r = w == 1u ? m : __umulhi(m, ml);
                b = (by0 + r) * (uint32_t)bins_x + bx0 + (m - r * w);
            }
            f(valid, qq, b, el);
        }
        q = qe;  // (a partial last step ends exactly at qe)
        k += 32;
        inc = n_inc;
        exc = n_exc;
        e = n_e;
    }
}

// Entry counts in sorted order (the scan input) and their exact u64 total.
__global__ void __launch_bounds__(256) bs_gather_kernel(const uint32_t* __restrict__ sval_sorted,
                                                        const uint32_t* __restrict__ tiles, uint32_t nsel,
                                                        uint32_t* __restrict__ out, unsigned long long* total) {
    __shared__ unsigned long long ws[8];
    const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
    uint32_t n = 0;
    if (k < nsel) {
        n = __ldg(tiles + __ldg(sval_sorted + k));
        out[k] = n;
    }
    const uint32_t w = __reduce_add_sync(FULL, n);  // <= 32 * 12288: no overflow
    if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = w;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long t = 0;
        for (int i = 0; i < 8; i++) t += ws[i];
        if (t) atomicAdd(total, t);
    }
}

// One warp: per-view sorted-element starts (the compaction's exclusive offsets at each view's
// first tile: selection is view-major and the depth sort keeps views apart), entry bases,
// segment table.
__global__ void bs_views_kernel(const uint32_t* __restrict__ sel_offsets, int tiles_per_view,
                                const uint32_t* __restrict__ offs, uint32_t nsel, int nv, uint32_t sege,
                                BsInfo* info) {
    const int lane = threadIdx.x;
    uint32_t start = nsel;
    if (lane < nv) start = lane == 0 ? 0u : sel_offsets[(size_t)lane * tiles_per_view];
    const uint32_t eb = start > 0 ? offs[start - 1] : 0u;  // entries before the view
    uint32_t ee = __shfl_down_sync(FULL, eb, 1);
    if (lane == nv - 1) ee = offs[nsel - 1];
    const uint32_t nseg = lane < nv ? (ee - eb + sege - 1) / sege : 0u;
    uint32_t inc = nseg;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(FULL, inc, o);
        if (lane >= o) inc += t;
    }
    if (lane < nv) {
        info->vstart[lane] = start;
        info->ebase[lane] = eb;
        info->segbase[lane] = inc - nseg;
    }
    if (lane == nv - 1) {
        info->vstart[nv] = nsel;
        info->ebase[nv] = ee;
        info->segbase[nv] = inc;
        info->sege = sege;
    }
}

__global__ void bs_count_kernel(const BsInfo* __restrict__ info, int nv, const uint32_t* __restrict__ offs,
                                const uint32_t* __restrict__ sval_sorted, const uint2* __restrict__ rect,
                                int bins_x, int nb, uint32_t* __restrict__ cnt, uint16_t* __restrict__ ebin,
                                uint32_t* __restrict__ eel) {
    extern __shared__ uint32_t bs_rows[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t seg = blockIdx.x * (blockDim.x >> 5) + warp;
    int v;
    uint32_t q0, q1;
    if (!bs_segment(info, nv, seg, v, q0, q1)) return;  // (no block-wide barriers below)
    uint32_t* row = bs_rows + (size_t)warp * nb;
    for (int b = lane; b < nb; b += 32) row[b] = 0u;
    const uint32_t k = bs_first_element(offs, info, v, q0);
    __syncwarp();
    bs_walk(k, info->vstart[v + 1], q0, q1, offs, sval_sorted, rect, bins_x,
            [&](bool valid, uint32_t qq, uint32_t b, uint32_t el) {
                if (valid) {
                    atomicAdd(row + b, 1u);
                    ebin[qq] = (uint16_t)b;  // the flattened entries, coalesced, for bs_scatter
                    eel[qq] = el;
                }
            });
    __syncwarp();
    uint32_t* out = cnt + (size_t)seg * nb;
    for (int b = lane; b < nb; b += 32) out[b] = row[b];
}

// grid (ceil(nb / 32), nv), 8 warps: lane = bin, warp w = the w-th eighth of the view's segments.
// The column of counts becomes its exclusive prefix; the bin's total goes to ranges[].y.
__global__ void __launch_bounds__(256) bs_colscan_kernel(const BsInfo* __restrict__ info, int nb,
                                                         uint32_t* __restrict__ cnt, uint2* __restrict__ ranges) {
    __shared__ uint32_t part[8][32];
    const int v = blockIdx.y, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int b = blockIdx.x * 32 + lane;
    const uint32_t s0 = info->segbase[v], s1 = info->segbase[v + 1];
    const uint32_t per = (s1 - s0 + 7) / 8;
    const uint32_t a0 = min(s1, s0 + warp * per), a1 = min(s1, a0 + per);
    uint32_t sum = 0;
    if (b < nb) {
#pragma unroll 8
        for (uint32_t s = a0; s < a1; s++) sum += cnt[(size_t)s * nb + b];
    }
    part[warp][lane] = sum;
    __syncthreads();
    uint32_t run = 0, tot = 0;
#pragma unroll
    for (int w = 0; w < 8; w++) {
        run += w < warp ? part[w][lane] : 0u;
        tot += part[w][lane];
    }
    if (b >= nb) return;
#pragma unroll 8
    for (uint32_t s = a0; s < a1; s++) {
        const uint32_t c = cnt[(size_t)s * nb + b];
        cnt[(size_t)s * nb + b] = run;
        run += c;
    }
    if (warp == 0) ranges[(size_t)v * nb + b] = make_uint2(0u, tot);
}

// one CTA of 1024 threads per view: ranges[v][b] = [base_v + excl_b, base_v + excl_b + total_b)
__global__ void __launch_bounds__(1024) bs_ranges_kernel(const BsInfo* __restrict__ info, int nb,
                                                         uint2* __restrict__ ranges) {
    typedef cub::BlockScan<uint32_t, 1024> Scan;
    __shared__ typename Scan::TempStorage tmp;
    const int v = blockIdx.x;
    const uint32_t base = info->ebase[v];
    uint2* R = ranges + (size_t)v * nb;
    const int per = (nb + 1023) / 1024;
    const int b0 = min(nb, (int)threadIdx.x * per), b1 = min(nb, b0 + per);
    uint32_t sum = 0;
    for (int b = b0; b < b1; b++) sum += R[b].y;
    uint32_t off, tot;
    Scan(tmp).ExclusiveSum(sum, off, tot);
    off += base;
    for (int b = b0; b < b1; b++) {
        const uint32_t c = R[b].y;
        R[b] = make_uint2(off, off + c);
        off += c;
    }
}

__global__ void bs_scatter_kernel(const BsInfo* __restrict__ info, int nv, int nb, const uint32_t* __restrict__ cnt,
                                  const uint2* __restrict__ ranges, const uint16_t* __restrict__ ebin,
                                  const uint32_t* __restrict__ eel, uint32_t* __restrict__ eval) {
    extern __shared__ uint32_t bs_rows[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t seg = blockIdx.x * (blockDim.x >> 5) + warp;
    int v;
    uint32_t q0, q1;
    if (!bs_segment(info, nv, seg, v, q0, q1)) return;
    uint32_t* row = bs_rows + (size_t)warp * nb;
    uint8_t* tag = reinterpret_cast<uint8_t*>(bs_rows + (size_t)(blockDim.x >> 5) * nb) + (size_t)warp * nb;
    const uint32_t* pre = cnt + (size_t)seg * nb;
    const uint2* R = ranges + (size_t)v * nb;
    for (int b = lane; b < nb; b += 32) row[b] = R[b].x + pre[b];
    __syncwarp();
    const unsigned lt = (1u << lane) - 1u;
    constexpr int U = 8;  // steps whose loads are issued together
    for (uint32_t q = q0; q < q1; q += 32 * U) {
        uint32_t bb[U], ee[U];
#pragma unroll
        for (int u = 0; u < U; u++) {
            const uint32_t qq = q + (uint32_t)(u * 32 + lane);
            bb[u] = qq < q1 ? (uint32_t)__ldg(ebin + qq) : 0xFFFFFFFFu;
            ee[u] = qq < q1 ? __ldg(eel + qq) : 0u;
        }
#pragma unroll
        for (int u = 0; u < U; u++) {
            // 32 consecutive entries of the flattened order; an element covers a bin once, so a
            // bin's earlier lanes are earlier elements: rank = earlier peers
            const uint32_t b = bb[u];
            const bool valid = b != 0xFFFFFFFFu;
            // common case: the step's bins are distinct (its entries are mostly a few elements'
            // rectangles) -- detected by a lane-id tag per bin, no warp match needed
            if (valid) tag[b] = (uint8_t)lane;
            __syncwarp();
            const bool own = !valid || tag[b] == (uint8_t)lane;
            if (__all_sync(FULL, own)) {
                if (valid) {
                    const uint32_t pos = row[b];
                    eval[pos] = ee[u];
                    row[b] = pos + 1u;
                }
            } else {
                const unsigned peers = __match_any_sync(FULL, b);
                const uint32_t pos = valid ? row[b] + (uint32_t)__popc(peers & lt) : 0u;
                __syncwarp();
                if (valid) {
                    eval[pos] = ee[u];
                    if (lane == 31 - __clz(peers)) row[b] = pos + 1u;  // the bin's last entry of this step
                }
            }
            __syncwarp();
        }
    }
}

int bs_warps_per_cta(int nb) {
    int w = (int)((96 * 1024) / ((size_t)nb * sizeof(uint32_t)));
    return std::max(1, std::min(BS_WARPS_MAX, w));
}

}  // namespace

// Entries per segment: BS_SEGE, or more for very large chunks, so that the segments (warps) stay
// about one resident wave and the [segment][bin] matrix stays small (the column scan reads it
// twice).
static int g_segment_override = 0;  // scoup_diag_set_binsort_segment

uint32_t binsort_segment_len(int64_t entries) {
    if (g_segment_override > 0) return (uint32_t)g_segment_override;
    const int64_t target = 148 * 48 * 16;  // (measured: longer segments cost the count and scatter more)
    const int64_t len = std::max<int64_t>(BS_SEGE, ((entries + target - 1) / target + 255) / 256 * 256);
    return (uint32_t)len;
}

void binsort_set_segment_override(int len) { g_segment_override = len > 0 ? (len + 31) / 32 * 32 : 0; }

size_t binsort_segments_max(int64_t entries, int nv) {
    const int64_t len = binsort_segment_len(entries);
    return (size_t)((entries + len - 1) / len + nv);
}

void launch_binsort_gather(const uint32_t* sval_sorted, const uint32_t* tiles, int64_t nsel, uint32_t* offs,
                           BsInfo* info, cudaStream_t s) {
    cudaMemsetAsync(&info->total, 0, sizeof(unsigned long long), s);
    bs_gather_kernel<<<(unsigned)((nsel + 255) / 256), 256, 0, s>>>(sval_sorted, tiles, (uint32_t)nsel, offs,
                                                                    &info->total);
}

void launch_binsort(const uint32_t* sel_offsets, int tiles_per_view, const uint32_t* offs,
                    const uint32_t* sval_sorted, const uint2* rect, int64_t nsel, int64_t entries, int nv,
                    int bins_x, int nb, BsInfo* info, uint32_t* cnt, uint16_t* ebin, uint32_t* eel, uint2* ranges,
                    uint32_t* eval, cudaStream_t s) {
    bs_views_kernel<<<1, 32, 0, s>>>(sel_offsets, tiles_per_view, offs, (uint32_t)nsel, nv,
                                     binsort_segment_len(entries), info);
    const int wpc = bs_warps_per_cta(nb);
    const size_t smem = (size_t)wpc * nb * sizeof(uint32_t);
    static size_t smem_set = 48 * 1024;
    if (smem > smem_set) {
        cudaFuncSetAttribute(bs_count_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        smem_set = smem;
    }
    const unsigned grid = (unsigned)((binsort_segments_max(entries, nv) + wpc - 1) / wpc);
    bs_count_kernel<<<grid, 32 * wpc, smem, s>>>(info, nv, offs, sval_sorted, rect, bins_x, nb, cnt, ebin, eel);
    bs_colscan_kernel<<<dim3((unsigned)((nb + 31) / 32), (unsigned)nv), 256, 0, s>>>(info, nb, cnt, ranges);
    bs_ranges_kernel<<<nv, 1024, 0, s>>>(info, nb, ranges);
    // (the scatter's rows plus a byte of lane tag per bin)
    const int wps = std::max(1, std::min(BS_WARPS_MAX, (int)((96 * 1024) / ((size_t)nb * 5))));
    const size_t smem_s = (size_t)wps * nb * 5;
    static size_t smem_set_s = 48 * 1024;
    if (smem_s > smem_set_s) {
        cudaFuncSetAttribute(bs_scatter_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_s);
        smem_set_s = smem_s;
    }
    const unsigned grid_s = (unsigned)((binsort_segments_max(entries, nv) + wps - 1) / wps);
    bs_scatter_kernel<<<grid_s, 32 * wps, smem_s, s>>>(info, nv, nb, cnt, ranges, ebin, eel, eval);
}

}  // namespace scoup
