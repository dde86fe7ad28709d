// kernels.cu -- per-Gaussian, binning and finalize kernels of the sm_100a path.
//
//   activate        DESIGN.md §3 G1: q/|q|, R(q), Sigma_3D = R diag(s)^2 R^T
//   preprocess      DESIGN.md §3 V1-V7: EWA projection, culls, support rect
//   depth pass, compactions   the depth chunks of a view batch (DESIGN.md §5 a3); the bin lists
//                   of a chunk are built in binsort.cu
//   ingest_codes    Algorithm 1's per-pixel TopK(W_v(p)) realised per region
//   topk            Eq. 6 Top-K + L1 renormalisation (Algorithm 1)
#include <cub/block/block_scan.cuh>

#include <climits>

#include <algorithm>

#include "internal.cuh"

namespace scoup {

namespace {

__device__ __forceinline__ float mul(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ float add(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ float sub(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ float dv(float a, float b) { return __fdiv_rn(a, b); }

inline unsigned grid_for(int64_t n, int block) {
    int64_t g = (n + block - 1) / block;
    return (unsigned)(g < 1 ? 1 : g);
}

// ------------------------------------------------------------------ activate (G1)
__global__ void activate_kernel(const float* __restrict__ means, const float* __restrict__ scales,
                                const float* __restrict__ rots, const float* __restrict__ opac,
                                int64_t G, PackedGaussians pg, ErrorLatch err) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= G) return;
    float mx = means[3 * i], my = means[3 * i + 1], mz = means[3 * i + 2];
    float s0 = scales[3 * i], s1 = scales[3 * i + 1], s2 = scales[3 * i + 2];
    float qw = rots[4 * i], qx = rots[4 * i + 1], qy = rots[4 * i + 2], qz = rots[4 * i + 3];
    float o = opac[i];
    bool ok = isfinite(mx) && isfinite(my) && isfinite(mz) && isfinite(qw) && isfinite(qx) &&
              isfinite(qy) && isfinite(qz) && isfinite(s0) && isfinite(s1) && isfinite(s2) &&
              s0 > 0.f && s1 > 0.f && s2 > 0.f && isfinite(o) && o >= 0.f && o <= 1.f;
    float n = __fsqrt_rn(add(add(add(mul(qw, qw), mul(qx, qx)), mul(qy, qy)), mul(qz, qz)));
    ok = ok && n > 0.f;
    if (!ok) {
        latch_error(err, ERR_GAUSSIAN, i);
        pg.a[i] = make_float4(0.f, 0.f, 0.f, -1.f);
        pg.b[i] = make_float4(0.f, 0.f, 0.f, 0.f);
        pg.c[i] = make_float2(0.f, 0.f);
        pg.s2[i] = 0.f;
        return;
    }
    float w = dv(qw, n), x = dv(qx, n), y = dv(qy, n), z = dv(qz, n);
    float R[3][3];
    R[0][0] = sub(1.f, mul(2.f, add(mul(y, y), mul(z, z))));
    R[0][1] = mul(2.f, sub(mul(x, y), mul(w, z)));
    R[0][2] = mul(2.f, add(mul(x, z), mul(w, y)));
    R[1][0] = mul(2.f, add(mul(x, y), mul(w, z)));
    R[1][1] = sub(1.f, mul(2.f, add(mul(x, x), mul(z, z))));
    R[1][2] = mul(2.f, sub(mul(y, z), mul(w, x)));
    R[2][0] = mul(2.f, sub(mul(x, z), mul(w, y)));
    R[2][1] = mul(2.f, add(mul(y, z), mul(w, x)));
    R[2][2] = sub(1.f, mul(2.f, add(mul(x, x), mul(y, y))));
    const float s[3] = {s0, s1, s2};
    float M[3][3];
#pragma unroll
    for (int a = 0; a < 3; a++)
#pragma unroll
        for (int b = 0; b < 3; b++) M[a][b] = mul(R[a][b], s[b]);
    float V[6];
    int k = 0;
#pragma unroll
    for (int a = 0; a < 3; a++)
#pragma unroll
        for (int b = a; b < 3; b++)
            V[k++] = add(add(mul(M[a][0], M[b][0]), mul(M[a][1], M[b][1])), mul(M[a][2], M[b][2]));
    pg.a[i] = make_float4(mx, my, mz, o);
    pg.b[i] = make_float4(V[0], V[1], V[2], V[3]);
    pg.c[i] = make_float2(V[4], V[5]);
    const float sm = fmaxf(s0, fmaxf(s1, s2));
    pg.s2[i] = sm * sm * 1.0001f;  // lambda_max(Sigma_3D), padded (GPU-only prune)
}

// ------------------------------------------------------------------ scene bounds
// Axis-aligned box of the valid means (init): the host derives each view batch's depth bound
// from it, hence how many bits the depth code needs.  Floats are mapped to order-preserving
// ints for atomicMin/Max.
__device__ __forceinline__ int ord_int(float f) {
    int b = __float_as_int(f);
    return b >= 0 ? b : b ^ 0x7FFFFFFF;
}

__global__ void bounds_kernel(PackedGaussians pg, int64_t G, int* bbox) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    int lo[3] = {INT_MAX, INT_MAX, INT_MAX}, hi[3] = {INT_MIN, INT_MIN, INT_MIN};
    for (; i < G; i += (int64_t)gridDim.x * blockDim.x) {
        const float4 A = pg.a[i];
        if (A.w < 0.f) continue;  // invalid Gaussian (latched at init)
        const int v[3] = {ord_int(A.x), ord_int(A.y), ord_int(A.z)};
#pragma unroll
        for (int a = 0; a < 3; a++) { lo[a] = min(lo[a], v[a]); hi[a] = max(hi[a], v[a]); }
    }
#pragma unroll
    for (int a = 0; a < 3; a++) {
        lo[a] = __reduce_min_sync(0xffffffffu, lo[a]);
        hi[a] = __reduce_max_sync(0xffffffffu, hi[a]);
    }
    if ((threadIdx.x & 31) == 0) {
#pragma unroll
        for (int a = 0; a < 3; a++) { atomicMin(bbox + a, lo[a]); atomicMax(bbox + 3 + a, hi[a]); }
    }
}

// ------------------------------------------------------------------ depth pass (V1, V2)
// Depth code of a visible Gaussian: bits(t_z) - bits(0.2f) >= 1 (positive floats order as their
// bit patterns, so codes order depths exactly; equal depths keep index order in the stable
// sorts).  Invisible: the all-ones code `none`.
__device__ __forceinline__ void camera_space(const float4& A, const Camera& cam, float t[3]) {
#pragma unroll
    for (int a = 0; a < 3; a++)
        t[a] = add(add(add(mul(cam.P[4 * a + 0], A.x), mul(cam.P[4 * a + 1], A.y)), mul(cam.P[4 * a + 2], A.z)),
                   cam.P[4 * a + 3]);
}

// Conservative screen-space reach of a Gaussian (GPU-only prune): with
// lambda_max(Sigma_3D) = s_max^2 and ||J W||_2 <= ||J||_F, the square support r of V7 is at most
// 3 sqrt(s_max^2 ||J||_F^2 + 0.3); padded for fp32 rounding.  mean2d is computed with the exact
// V3 operations, so it equals preprocess's.
// The same bound with hardware reciprocal / square root (the depth pass's hot path): their few-ulp
// errors move mean2d by < 1e-6 |fx u| px and the radius by < 1e-6 relative, inside the bound's
// 0.2% + 1 px padding, which a second 1e-5 |fx u| + 1e-5 |fy v| term widens further.
__device__ __forceinline__ void reach_fast(const float t[3], float s2max, const Camera& cam, float& mx, float& my,
                                           float& rb) {
    const float iz = __fdividef(1.0f, t[2]);
    const float u = t[0] * iz, v = t[1] * iz;
    const float fu = cam.fx * u, fv = cam.fy * v;
    mx = fu + cam.cx;
    my = fv + cam.cy;
    const float jf2 = (cam.fx * cam.fx * (1.0f + u * u) + cam.fy * cam.fy * (1.0f + v * v)) * iz * iz;
    float sq;
    asm("sqrt.approx.f32 %0, %1;" : "=f"(sq) : "f"(s2max * jf2 + K_LOWPASS));
    rb = 3.0f * sq * 1.002f + 1.0f + 1e-5f * (fabsf(fu) + fabsf(fv));
}
// Stable compactions over the batch indices (below) and the depth pass share one tiling: tiles of
// SEL_TILE Gaussians per view, 8 warps each owning SEL_ITEMS rounds of 32 consecutive Gaussians.
constexpr int SEL_ITEMS = 16;
constexpr int SEL_TILE = 256 * SEL_ITEMS;

// Packed reach box in 16x16 tiles for the far-chunk predicate (x0 | x1 << 8 | y0 << 16 | y1 << 24;
// x0 > x1: no tile); images up to 255 tiles a side (wider ones recompute in the far predicate).
constexpr uint32_t TRECT_EMPTY = 0x000000FFu;

// The depth pass's camera: the rows of [R|t], the focal lengths and their squares, and the
// principal point in tile units ((c - 0.5) / 16), last tile indices.
struct DepthCam {
    float P[12];
    float fx, fy, fx2, fy2, cxt, cyt;
    int tx1, ty1;
};
__device__ __forceinline__ DepthCam depth_cam(const Camera& cam) {
    DepthCam d;
#pragma unroll
    for (int k = 0; k < 12; k++) d.P[k] = cam.P[k];
    d.fx = cam.fx;
    d.fy = cam.fy;
    d.fx2 = cam.fx * cam.fx;
    d.fy2 = cam.fy * cam.fy;
    d.cxt = (cam.cx - 0.5f) * (1.0f / TILE);
    d.cyt = (cam.cy - 0.5f) * (1.0f / TILE);
    d.tx1 = (cam.width + TILE - 1) / TILE - 1;
    d.ty1 = (cam.height + TILE - 1) / TILE - 1;
    return d;
}

// Depth code of Gaussian i in the view (V1, V2, the conservative on-screen test) and, when
// visible, its packed reach box in 16x16 tiles.  The reach is reach_fast's bound (same terms, with
// FMAs; its 0.2% + 1 px padding is far above their few-ulp differences), taken in tile units: the
// tiles whose pixel centres x + 0.5 can lie within [mx - rb, mx + rb] are
// floor((mx -+ rb - 0.5) / 16) = floor(fu / 16 + (cx - 0.5) / 16 -+ rb / 16) (cvt.rmi saturates:
// out-of-range and infinite bounds clamp like the exact floor would).  Visible: the box clamped to
// the image's tile grid is non-empty (a pixel centre of the grid lies within the reach) -- a
// conservative superset of the pixels the exact EWA support can reach.  t[2] (the depth code) is
// computed with the exact V1 operations.
__device__ __forceinline__ uint32_t depth_code(const float4& A, float s2, const DepthCam& dc, uint32_t none,
                                               uint32_t& rect, bool& beyond) {
    uint32_t c = none;
    rect = TRECT_EMPTY;
    beyond = false;
    float t[3];
#pragma unroll
    for (int a = 0; a < 3; a++)
        t[a] = add(add(add(mul(dc.P[4 * a + 0], A.x), mul(dc.P[4 * a + 1], A.y)), mul(dc.P[4 * a + 2], A.z)),
                   dc.P[4 * a + 3]);
    if (t[2] > K_NEAR && A.w >= K_AMIN) {
        const float iz = __fdividef(1.0f, t[2]);
        const float u = t[0] * iz, v = t[1] * iz;
        const float fu = dc.fx * u, fv = dc.fy * v;
        const float jf2 = fmaf(dc.fx2, fmaf(u, u, 1.0f), dc.fy2 * fmaf(v, v, 1.0f)) * (iz * iz);
        float sq;
        asm("sqrt.approx.f32 %0, %1;" : "=f"(sq) : "f"(fmaf(s2, jf2, K_LOWPASS)));
        const float rb = fmaf(3.006f, sq, fmaf(1e-5f, fabsf(fu) + fabsf(fv), 1.0f));
        const float rt = rb * (1.0f / TILE);
        const float ax = fmaf(fu, 1.0f / TILE, dc.cxt), ay = fmaf(fv, 1.0f / TILE, dc.cyt);
        const int x0 = max(0, __float2int_rd(ax - rt)), x1 = min(dc.tx1, __float2int_rd(ax + rt));
        const int y0 = max(0, __float2int_rd(ay - rt)), y1 = min(dc.ty1, __float2int_rd(ay + rt));
        if (x0 <= x1 && y0 <= y1) {
            c = __float_as_uint(t[2]) - __float_as_uint(K_NEAR);
            if (!(c < none)) {  // beyond the host's depth bound for the batch (cannot happen)
                beyond = true;
                c = none;
            } else {
                rect = (uint32_t)x0 | ((uint32_t)x1 << 8) | ((uint32_t)y0 << 16) | ((uint32_t)y1 << 24);
            }
        }
    }
    return c;
}

// The split histogram (DESIGN.md §5 a3): the codes' top HIST_BITS bits of every HIST_SAMPLE-th
// Gaussian per view (the split is a heuristic -- any threshold is exact -- and the near count
// comes from the compaction).  One thread per sampled (view, Gaussian).
__global__ void __launch_bounds__(256) depth_hist_kernel(PackedGaussians pg, int64_t G, const CamBatch cams,
                                                         int key_bits, uint32_t* __restrict__ hist) {
    __shared__ uint32_t sh[NHIST];
    for (int k = threadIdx.x; k < NHIST; k += blockDim.x) sh[k] = 0;
    __syncthreads();
    const int view = blockIdx.y;
    const DepthCam dc = depth_cam(cams.cam[view]);
    const uint32_t none = (1u << key_bits) - 1u;
    const int shift = key_bits > HIST_BITS ? key_bits - HIST_BITS : 0;
    const int64_t n = (G + HIST_SAMPLE - 1) / HIST_SAMPLE;
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = k * HIST_SAMPLE;
        uint32_t rect;
        bool beyond;
        const uint32_t c = depth_code(pg.a[i], pg.s2[i], dc, none, rect, beyond);
        if (c != none) atomicAdd(&sh[c >> shift], 1u);
    }
    __syncthreads();
    for (int k = threadIdx.x; k < NHIST; k += blockDim.x)
        if (sh[k]) atomicAdd(&hist[view * NHIST + k], sh[k]);
}

// One thread per Gaussian and all views of the batch, grid (tiles of SEL_TILE Gaussians): writes
// code[j] (j = v*G + i) and the packed reach box, counts the visible Gaussians, and runs the count
// pass of the near chunk's stable compaction in the same sweep (code < thr[v]: the predicate words
// and per-(view, tile) counts sel_scan / sel_scatter take, laid out as sel_count_kernel's).
// Off-screen Gaussians (conservative reach misses the image) are invisible.  Each Gaussian is read
// once per batch (groups of DP_GROUP items held in registers while the views loop, each camera
// loaded once per group).  The far chunk's predicate reads only the reach box, so the box of an
// invisible or near element is written empty (it can never be a far element).
constexpr int DP_GROUP = 4;
__global__ void __launch_bounds__(256) depth_pass_kernel(PackedGaussians pg, int64_t G, const CamBatch cams,
                                                         int key_bits, const uint32_t* __restrict__ thr,
                                                         uint32_t* __restrict__ code,
                                                         unsigned long long* visible_ctr, ErrorLatch err, int tiles_x,
                                                         int tiles_y, uint32_t* __restrict__ trect,
                                                         uint32_t* __restrict__ counts, uint32_t* __restrict__ bits) {
    __shared__ uint32_t sbits[MAX_VB][8][SEL_ITEMS];  // predicate words (view, warp, item)
    __shared__ uint32_t sn[MAX_VB][8];                // near counts (view, warp)
    __shared__ uint32_t sthr[MAX_VB], wv[8];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nv = cams.n;
    const uint32_t none = (1u << key_bits) - 1u;
    if (threadIdx.x < nv) sthr[threadIdx.x] = thr[threadIdx.x];
    if (lane < nv) sn[lane][warp] = 0u;
    __syncthreads();
    const int64_t base = (int64_t)blockIdx.x * SEL_TILE + warp * (SEL_ITEMS * 32) + lane;
    const int nit = (int)max((int64_t)0, min((int64_t)SEL_ITEMS, (G - base + 31) / 32));  // items with i < G
    uint32_t nvis = 0;
    for (int g = 0; g < SEL_ITEMS; g += DP_GROUP) {
        float4 A[DP_GROUP];
        float s2[DP_GROUP];
#pragma unroll
        for (int u = 0; u < DP_GROUP; u++) {
            if (g + u < nit) {
                A[u] = pg.a[base + 32 * (g + u)];
                s2[u] = pg.s2[base + 32 * (g + u)];
            } else {
                A[u] = make_float4(0.f, 0.f, 0.f, -1.f);  // (fails the opacity test: invisible)
                s2[u] = 0.f;
            }
        }
        for (int v = 0; v < nv; v++) {
            const DepthCam dc = depth_cam(cams.cam[v]);  // (warp-uniform: one register copy per group)
            const uint32_t tv = sthr[v];
            const int64_t j0 = (int64_t)v * G + base;
            uint32_t nn = 0;  // near elements of the warp's items in this group
#pragma unroll
            for (int u = 0; u < DP_GROUP; u++) {
                const int it = g + u;
                uint32_t rect;
                bool beyond;
                const uint32_t c = depth_code(A[u], s2[u], dc, none, rect, beyond);
                const bool near = c < tv;  // (tv <= none: the invisible code is never near)
                if (it < nit) {
                    if (beyond) latch_error(err, ERR_DEPTHKEY, j0 + 32 * it);
                    code[j0 + 32 * it] = c;
                    if (trect) trect[j0 + 32 * it] = near ? TRECT_EMPTY : rect;  // (rect is empty when invisible)
                    nvis += c != none ? 1u : 0u;
                }
                const unsigned b = __ballot_sync(0xffffffffu, near);
                if (lane == 0) sbits[v][warp][it] = b;
                nn += (uint32_t)__popc(b);
            }
            if (lane == 0) sn[v][warp] += nn;
        }
    }
    nvis = __reduce_add_sync(0xffffffffu, nvis);
    if (lane == 0) wv[warp] = nvis;
    __syncthreads();
    // the (view, tile) predicate words and counts: tile = v * gridDim.x + blockIdx.x
    for (int k = threadIdx.x; k < nv * 8 * SEL_ITEMS; k += blockDim.x) {
        const int v = k / (8 * SEL_ITEMS), r = k - v * (8 * SEL_ITEMS);
        bits[((int64_t)v * gridDim.x + blockIdx.x) * (8 * SEL_ITEMS) + r] = (&sbits[v][0][0])[r];
    }
    if (threadIdx.x < nv) {
        uint32_t tot = 0;
#pragma unroll
        for (int w = 0; w < 8; w++) tot += sn[threadIdx.x][w];
        counts[(int64_t)threadIdx.x * gridDim.x + blockIdx.x] = tot;
    }
    if (threadIdx.x == 0) {
        uint32_t vis = 0;
#pragma unroll
        for (int w = 0; w < 8; w++) vis += wv[w];
        if (vis) atomicAdd(visible_ctr, (unsigned long long)vis);
    }
}

// ------------------------------------------------------------------ chunk selection
// Near chunk of view v: codes below thr[v].  Far chunk: the other visible codes whose
// conservative reach touches a tile that is still live after the near chunk.  Both are stable
// compactions over the batch indices (below), so index order is kept.

// Summed-area table of the live tiles of each view: sat[v][(ty+1)*(tx_n+1) + tx+1] = number of
// live tiles in [0, tx] x [0, ty] (< 2^16: at most MAX_SAT_ENTRIES tiles).  One block per view;
// rows then columns, in shared memory.

__global__ void __launch_bounds__(1024) live_sat_kernel(const uint8_t* __restrict__ tile_live, int tiles_x,
                                                        int tiles_y, uint16_t* __restrict__ sat) {
    __shared__ uint32_t S[MAX_SAT_ENTRIES];
    const int v = blockIdx.x;
    const int W1 = tiles_x + 1, H1 = tiles_y + 1;
    const uint8_t* lv = tile_live + (int64_t)v * tiles_x * tiles_y;
    for (int k = threadIdx.x; k < W1 * H1; k += blockDim.x) {
        const int x = k % W1, y = k / W1;
        S[k] = (x > 0 && y > 0) ? (uint32_t)lv[(y - 1) * tiles_x + (x - 1)] : 0u;
    }
    __syncthreads();
    for (int y = threadIdx.x; y < H1; y += blockDim.x)
        for (int x = 1; x < W1; x++) S[y * W1 + x] += S[y * W1 + x - 1];
    __syncthreads();
    for (int x = threadIdx.x; x < W1; x += blockDim.x)
        for (int y = 1; y < H1; y++) S[y * W1 + x] += S[(y - 1) * W1 + x];
    __syncthreads();
    for (int k = threadIdx.x; k < W1 * H1; k += blockDim.x) sat[(int64_t)v * W1 * H1 + k] = (uint16_t)S[k];
}

// ------------------------------------------------------------------ stable compaction
// The chunk selections as one stable compaction over the batch indices j = v * G + i (index order
// kept, so equal depth codes keep index order through the stable depth sort):
// count per 4096-element tile -> exclusive scan of the tile counts (one CTA) -> scatter.  Each
// warp owns 512 consecutive elements of its tile (16 rounds of 32), so ranks are ballot prefix
// sums in order.  Predicates: the near chunk (code below the view's split), the far chunk (code
// at or beyond the split and the conservative reach box covering a live tile).

struct FarSel {
    const uint32_t* code;
    const uint32_t* thr;
    int64_t G;
    uint32_t none;
    const uint32_t* trect;   // packed boxes from the depth pass, or NULL: recompute
    const uint16_t* sat;     // live-tile summed-area tables
    int tiles_x, tiles_y;
    PackedGaussians pg;
    const CamBatch* cams;    // device copy (recompute path)
    // With packed boxes only the box is loaded: the depth pass wrote it empty for invisible and
    // near elements, so a non-empty box is a visible code at or beyond the split.  Loads are
    // unconditional (coalesced; the branch-free loads of a thread's items can all be in flight).
    __device__ __forceinline__ uint2 load(int view, int64_t i) const {
        const int64_t j = (int64_t)view * G + i;
        return trect ? make_uint2(0u, trect[j]) : make_uint2(code[j], 0u);
    }
    __device__ __forceinline__ bool test(int view, int64_t i, uint2 v) const {
        int x0, x1, y0, y1;
        if (trect) {
            const uint32_t r = v.y;
            x0 = (int)(r & 255u); x1 = (int)((r >> 8) & 255u); y0 = (int)((r >> 16) & 255u); y1 = (int)(r >> 24);
        } else {
            const uint32_t c = v.x;
            if (c == none || c < thr[view]) return false;
            const Camera& cam = cams->cam[view];
            float t[3];
            camera_space(pg.a[i], cam, t);
            float mx, my, rb;
            reach_fast(t, pg.s2[i], cam, mx, my, rb);
            x0 = max(0, (int)floorf((mx - rb - 0.5f) * (1.0f / TILE)));
            x1 = min(tiles_x - 1, (int)floorf((mx + rb - 0.5f) * (1.0f / TILE)));
            y0 = max(0, (int)floorf((my - rb - 0.5f) * (1.0f / TILE)));
            y1 = min(tiles_y - 1, (int)floorf((my + rb - 0.5f) * (1.0f / TILE)));
        }
        if (x0 > x1 || y0 > y1) return false;
        const int W1 = tiles_x + 1;
        const uint16_t* S = ssat;  // the view's table, staged in shared memory by the kernel
        const int n = (int)S[(y1 + 1) * W1 + x1 + 1] - (int)S[y0 * W1 + x1 + 1] - (int)S[(y1 + 1) * W1 + x0] +
                      (int)S[y0 * W1 + x0];
        return n > 0;
    }
    const uint16_t* ssat = nullptr;
    static constexpr bool kStageSat = true;
};

// Blocks stride over the tiles of their view (gridDim.x blocks per view), so the far predicate's
// table is staged into shared memory once per block, not once per tile.
template <class Pred>
__global__ void __launch_bounds__(256) sel_count_kernel(Pred pred, int64_t G, int tiles_per_view,
                                                        uint32_t* __restrict__ counts, uint32_t* __restrict__ bits) {
    __shared__ uint32_t ws[2][8];
    extern __shared__ uint16_t sat_sh[];  // the far predicate's live-tile table of this view
    const int view = blockIdx.y, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (Pred::kStageSat) {
        const int n = (pred.tiles_x + 1) * (pred.tiles_y + 1);
        const uint16_t* S = pred.sat + (int64_t)view * n;
        for (int k = threadIdx.x; k < n; k += blockDim.x) sat_sh[k] = S[k];
        pred.ssat = sat_sh;
        __syncthreads();
    }
    int pb = 0;
    for (int tl = blockIdx.x; tl < tiles_per_view; tl += gridDim.x, pb ^= 1) {
        const int64_t base = (int64_t)tl * SEL_TILE + warp * (SEL_ITEMS * 32) + lane;
        const int64_t tile = (int64_t)view * tiles_per_view + tl;
        uint32_t n = 0, word = 0;
        uint2 v[SEL_ITEMS];
#pragma unroll
        for (int it = 0; it < SEL_ITEMS; it++) {  // every load of the tile first
            const int64_t i = base + it * 32;
            v[it] = i < G ? pred.load(view, i) : make_uint2(0xFFFFFFFFu, 0u);
        }
#pragma unroll
        for (int it = 0; it < SEL_ITEMS; it++) {
            const int64_t i = base + it * 32;
            const unsigned b = __ballot_sync(0xffffffffu, i < G && pred.test(view, i, v[it]));
            n += __popc(b);
            if (lane == it) word = b;  // the warp's 16 predicate words, one per lane, for the scatter
        }
        if (lane < SEL_ITEMS) bits[(tile * 8 + warp) * SEL_ITEMS + lane] = word;
        if (lane == 0) ws[pb][warp] = n;  // (double-buffered: one barrier per tile)
        __syncthreads();
        if (threadIdx.x == 0) {
            uint32_t tot = 0;
#pragma unroll
            for (int w = 0; w < 8; w++) tot += ws[pb][w];
            counts[tile] = tot;
        }
    }
}

// exclusive scan of n tile counts in place (one CTA of 1024 threads, n <= 1024 * 64); total -> *nsel
__global__ void __launch_bounds__(1024) sel_scan_kernel(uint32_t* __restrict__ counts, int n, int* __restrict__ nsel) {
    typedef cub::BlockScan<uint32_t, 1024> Scan;
    __shared__ typename Scan::TempStorage tmp;
    const int per = (n + 1023) / 1024;
    const int b0 = min(n, threadIdx.x * per), b1 = min(n, b0 + per);
    uint32_t sum = 0;
    for (int k = b0; k < b1; k++) sum += counts[k];
    uint32_t off, total;
    Scan(tmp).ExclusiveSum(sum, off, total);
    for (int k = b0; k < b1; k++) {
        const uint32_t c = counts[k];
        counts[k] = off;
        off += c;
    }
    if (threadIdx.x == 0) *nsel = (int)total;
}

// scatter from the count pass's predicate words (no second evaluation of the predicate)
__global__ void __launch_bounds__(256) sel_scatter_kernel(int64_t G, const uint32_t* __restrict__ offsets,
                                                          const uint32_t* __restrict__ bits, uint32_t* __restrict__ sel) {
    __shared__ uint32_t ws[8];
    const int view = blockIdx.y, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t base = (int64_t)blockIdx.x * SEL_TILE + warp * (SEL_ITEMS * 32) + lane;
    const int64_t tile = (int64_t)view * gridDim.x + blockIdx.x;
    const uint32_t word = lane < SEL_ITEMS ? bits[(tile * 8 + warp) * SEL_ITEMS + lane] : 0u;
    const uint32_t tot = __reduce_add_sync(0xffffffffu, (uint32_t)__popc(word));
    if (lane == 0) ws[warp] = tot;
    __syncthreads();
    uint32_t run = offsets[tile];
    for (int w = 0; w < warp; w++) run += ws[w];
    const unsigned lt = (1u << lane) - 1u;
#pragma unroll
    for (int it = 0; it < SEL_ITEMS; it++) {
        const unsigned b = __shfl_sync(0xffffffffu, word, it);
        if ((b >> lane) & 1u) sel[run + __popc(b & lt)] = (uint32_t)((int64_t)view * G + base + it * 32);
        run += __popc(b);
    }
}

// counts: [tiles] tile counts, then [tiles * 128] predicate words (select_counts_needed)
template <class Pred>
static void compact(const Pred& pred, int64_t G, int nviews, uint32_t* counts, uint32_t* sel, int* nsel,
                    cudaStream_t s) {
    const dim3 grid(grid_for(G, SEL_TILE), (unsigned)nviews);
    const int64_t tiles = (int64_t)grid.x * grid.y;
    uint32_t* bits = counts + tiles;
    const size_t smem = Pred::kStageSat ? sizeof(uint16_t) * (pred.tiles_x + 1) * (pred.tiles_y + 1) : 0;
    if (smem > 48 * 1024)
        cudaFuncSetAttribute(sel_count_kernel<Pred>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    // (the far predicate: one resident wave of blocks, each staging its view's table once)
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (sms <= 0) sms = 148;
    }
    const unsigned per_view = (unsigned)std::max(1, (sms * 8) / std::max(1, nviews));
    const dim3 cgrid(Pred::kStageSat ? std::min<unsigned>(grid.x, per_view) : grid.x, (unsigned)nviews);
    sel_count_kernel<Pred><<<cgrid, 256, smem, s>>>(pred, G, (int)grid.x, counts, bits);
    sel_scan_kernel<<<1, 1024, 0, s>>>(counts, (int)tiles, nsel);
    sel_scatter_kernel<<<grid, 256, 0, s>>>(G, counts, bits, sel);
}

// ------------------------------------------------------------------ preprocess (V2-V7)
// One thread per selected element e (batch index j = sel[e], view v = j / G, Gaussian i): the EWA
// records at e (compact), the bin count of the support rectangle, and the sort pair
// ((v << key_bits) | code, e).
__global__ void __launch_bounds__(256) preprocess_kernel(PackedGaussians pg, int64_t G, const CamBatch cams,
                                                         Binning bn, ViewBuffers vb, int key_bits,
                                                         const uint32_t* __restrict__ sel, int64_t nsel,
                                                         uint32_t* __restrict__ skey, uint32_t* __restrict__ sval) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= nsel) return;  // (no block-wide barrier below)
    const uint32_t j = sel[e];
    const int view = (int)(j / G);
    const int64_t i = (int64_t)j - (int64_t)view * G;
    const Camera& cam = cams.cam[view];
    // The element's gathers (Gaussian record, depth code) as 16-byte asynchronous copies into
    // the thread's own shared-memory slots: they bypass L1, so the kernel keeps its loads in
    // flight when it runs next to resident raster CTAs whose carveout leaves almost no L1
    // (measured: 72 -> 130 us per launch with the maximum shared-memory carveout otherwise).
    __shared__ float4 g_a[256], g_b[256], g_c[256];
    __shared__ uint4 g_k[256];
    {
        const int t_ = threadIdx.x;
        auto cp16 = [](void* dst, const void* src) {
            const uint32_t sa = (uint32_t)__cvta_generic_to_shared(dst);
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(src));
        };
        cp16(&g_a[t_], pg.a + i);
        cp16(&g_b[t_], pg.b + i);
        cp16(&g_c[t_], reinterpret_cast<const float4*>(pg.c) + (i >> 1));  // the aligned pair holding c[i]
        cp16(&g_k[t_], reinterpret_cast<const uint4*>(vb.code) + (j >> 2));   // the aligned 4 codes holding code[j]
        asm volatile("cp.async.commit_group;\n" ::);
        asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    }
    {
        const float4 A = g_a[threadIdx.x];
        uint32_t ntiles = 0;
        const float o = A.w;
        float t[3];
        camera_space(A, cam, t);
        // V2: near plane; exact opacity cull (alpha <= o < 1/255 never contributes)
        if (t[2] > K_NEAR && o >= K_AMIN) {
            float4 B = g_b[threadIdx.x];
            const float4 C4 = g_c[threadIdx.x];
            float2 Cc = (i & 1) ? make_float2(C4.z, C4.w) : make_float2(C4.x, C4.y);
            const float Vm[3][3] = {{B.x, B.y, B.z}, {B.y, B.w, Cc.x}, {B.z, Cc.x, Cc.y}};
            // V3
            float u = dv(t[0], t[2]), v = dv(t[1], t[2]);
            float mx = add(mul(cam.fx, u), cam.cx);
            float my = add(mul(cam.fy, v), cam.cy);
            float j00 = dv(cam.fx, t[2]);
            float j02 = dv(-mul(cam.fx, u), t[2]);
            float j11 = dv(cam.fy, t[2]);
            float j12 = dv(-mul(cam.fy, v), t[2]);
            // V4: Q = J W
            float Q[2][3];
#pragma unroll
            for (int b = 0; b < 3; b++) {
                Q[0][b] = add(mul(j00, cam.P[0 * 4 + b]), mul(j02, cam.P[2 * 4 + b]));
                Q[1][b] = add(mul(j11, cam.P[1 * 4 + b]), mul(j12, cam.P[2 * 4 + b]));
            }
            // V5: U = Q Sigma_3D;  Sigma_2D = U Q^T + 0.3 I
            float U[2][3];
#pragma unroll
            for (int a = 0; a < 2; a++)
#pragma unroll
                for (int b = 0; b < 3; b++)
                    U[a][b] = add(add(mul(Q[a][0], Vm[0][b]), mul(Q[a][1], Vm[1][b])), mul(Q[a][2], Vm[2][b]));
            float sxx = add(add(add(mul(U[0][0], Q[0][0]), mul(U[0][1], Q[0][1])), mul(U[0][2], Q[0][2])), K_LOWPASS);
            float sxy = add(add(mul(U[0][0], Q[1][0]), mul(U[0][1], Q[1][1])), mul(U[0][2], Q[1][2]));
            float syy = add(add(add(mul(U[1][0], Q[1][0]), mul(U[1][1], Q[1][1])), mul(U[1][2], Q[1][2])), K_LOWPASS);
            // V6: conic
            float det = sub(mul(sxx, syy), mul(sxy, sxy));
            if (det > 0.f) {
                float ca = dv(syy, det), cb = dv(-sxy, det), cc = dv(sxx, det);
                // V7: radius of the square support
                float mid = mul(0.5f, add(sxx, syy));
                float lam = add(mid, __fsqrt_rn(fmaxf(0.f, sub(mul(mid, mid), det))));
                float r = mul(3.f, __fsqrt_rn(lam));
                float qa = mul(ca, K_HALF_LOG2E), qb = mul(cb, K_LOG2E_NEG), qc = mul(cc, K_HALF_LOG2E);
                // GPU-only conservative prune (not part of the spec):
                // y < ycut  =>  o * exp2_spec(y) < 1/255 with a 0.7% margin.
                float ycut = -log2f(255.f * o) - 0.01f;
                // support = square |d| <= r intersected with the bbox of the alpha >= 1/255
                // ellipse d^T conic d <= m^2, m^2 = -2 ln2 ycut.  The bbox half-widths are
                // m sqrt((conic^-1)_xx), taken from the conic actually evaluated (fp64, so
                // an ill-conditioned det cannot shrink it) and padded; exact test per pixel.
                float hx = r, hy = r;
                {
                    // The pixel's fp32 q has absolute error ~ eps * (size of its terms), which for
                    // far off-screen near-plane Gaussians is not negligible: widen the level set by
                    // 1e-6 * (bound on the terms over the current box), twice.
                    double dca = ca, dcb = cb, dcc = cc;
                    double detc = dca * dcc - dcb * dcb;
                    if (detc > 0.0) {
                        // half-widths m sqrt((conic^-1)_xx), m sqrt((conic^-1)_yy): the square
                        // roots of the inverse's diagonal once, sqrt(m^2) per round (fp64
                        // rounding far inside the 1.001 and +0.01 margins)
                        const double inv = 1.0 / detc;
                        const double sxx = sqrt(dcc * inv), syy = sqrt(dca * inv);
                        const double kx = fabs((double)qa) + 0.5 * fabs((double)qb);
                        const double ky = fabs((double)qc) + 0.5 * fabs((double)qb);
                        double yc = (double)ycut;
                        double ex = r, ey = r;
                        for (int it = 0; it < 3; it++) {
                            double m2 = -2.0 * 0.6931471805599453 * yc;
                            if (m2 <= 0.0) break;
                            const double m = sqrt(m2);
                            ex = fmin((double)r, m * sxx * 1.001 + 0.01);
                            ey = fmin((double)r, m * syy * 1.001 + 0.01);
                            double mq = kx * ex * ex + ky * ey * ey;
                            yc = (double)ycut - 0.01 - 2e-6 * mq;
                        }
                        hx = (float)ex;
                        hy = (float)ey;
                    }
                }
                float padx = 1.0f + 1e-6f * (fabsf(mx) + hx);
                float pady = 1.0f + 1e-6f * (fabsf(my) + hy);
                float fx0 = floorf(mx - hx - 0.5f - padx), fx1 = ceilf(mx + hx - 0.5f + padx);
                float fy0 = floorf(my - hy - 0.5f - pady), fy1 = ceilf(my + hy - 0.5f + pady);
                const float Wm1 = (float)(cam.width - 1), Hm1 = (float)(cam.height - 1);
                bool finite = isfinite(mx) && isfinite(my) && isfinite(r) && isfinite(qa) && isfinite(qb) && isfinite(qc);
                if (finite && fx1 >= 0.f && fx0 <= Wm1 && fy1 >= 0.f && fy0 <= Hm1) {
                    int x0 = (int)fmaxf(fx0, 0.f), x1 = (int)fminf(fx1, Wm1);
                    int y0 = (int)fmaxf(fy0, 0.f), y1 = (int)fminf(fy1, Hm1);
                    int tx0 = x0 >> bn.bshx, tx1 = (x1 >> bn.bshx) + 1, ty0 = y0 >> bn.bshy, ty1 = (y1 >> bn.bshy) + 1;
                    ntiles = (uint32_t)((tx1 - tx0) * (ty1 - ty0));
                    const float4 r0 = make_float4(mx, my, r, o), r1 = make_float4(qa, qb, qc, ycut);
                    const float2 ext = make_float2(hx + padx, hy + pady);
                    const Span sp = span_setup(r0, r1, ext);
                    vb.rect[e] = make_uint2((uint32_t)tx0 | ((uint32_t)ty0 << 16), (uint32_t)tx1 | ((uint32_t)ty1 << 16));
                    vb.rec0[e] = r0;
                    vb.rec1[e] = r1;
                    vb.rec2[e] = make_float4(ext.x, ext.y, __uint_as_float((uint32_t)i), sp.sy);
                    vb.rec3[e] = make_float4(sp.ky * sp.ia, sp.yc * sp.ia, sp.cq, sp.box_only ? -1.f : sp.sx);
                }
            }
        }
        vb.tiles[e] = ntiles;
        const uint4 k4 = g_k[threadIdx.x];
        const uint32_t kq = j & 3u;
        skey[e] = ((uint32_t)view << key_bits) | (kq == 0 ? k4.x : kq == 1 ? k4.y : kq == 2 ? k4.z : k4.w);
        sval[e] = (uint32_t)e;
    }
}

// ------------------------------------------------------------------ ingest dense features
// Dense region features (Eq. 3, the dense-uplift baseline): copy, finite check only.
__global__ void ingest_dense_kernel(const float* __restrict__ in, int64_t n, float* __restrict__ out, ErrorLatch err) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    float v = in[k];
    if (!isfinite(v)) {
        latch_error(err, ERR_CODE, k);
        v = 0.f;
    }
    out[k] = v;
}

// ------------------------------------------------------------------ ingest codes
// Validate each region code and truncate it to its K largest slots (ties -> lower atom),
// Algorithm 1's per-pixel TopK(W_v(p)).  No renormalisation.
__global__ void ingest_codes_kernel(const uint32_t* __restrict__ atoms_in, const float* __restrict__ coefs_in,
                                    int64_t rows, int S, int K, int L, uint32_t* __restrict__ atoms_out,
                                    float* __restrict__ coefs_out, ErrorLatch err) {
    int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= rows) return;
    uint32_t a[MAX_S];
    float c[MAX_S];
    for (int s = 0; s < S; s++) {
        a[s] = atoms_in[r * S + s];
        c[s] = coefs_in[r * S + s];
        if (a[s] != NONE && (a[s] >= (uint32_t)L || !isfinite(c[s]) || c[s] < 0.f)) {
            latch_error(err, ERR_CODE, r * S + s);
            a[s] = NONE;
            c[s] = 0.f;
        }
    }
    if (S > K) {
        for (int kept = 0; kept < K; kept++) {
            int best = -1;
            for (int s = kept; s < S; s++) {
                if (a[s] == NONE) continue;
                if (best < 0 || c[s] > c[best] || (c[s] == c[best] && a[s] < a[best])) best = s;
            }
            if (best < 0) break;
            uint32_t ta = a[kept]; float tc = c[kept];
            a[kept] = a[best]; c[kept] = c[best];
            a[best] = ta; c[best] = tc;
        }
        for (int s = K; s < S; s++) { a[s] = NONE; c[s] = 0.f; }
    }
    for (int s = 0; s < S; s++) {
        atoms_out[r * S + s] = a[s];
        coefs_out[r * S + s] = c[s];
    }
}

// ------------------------------------------------------------------ Top-K (Eq. 6)
// One thread per Gaussian row.  The KMAX best (value, atom) pairs live in registers,
// ordered (value desc, atom asc); a new value enters only if strictly larger than the current
// KMAX-th and is shift-inserted after every equal value (atoms are scanned ascending), so ties
// keep the lower atom.
// Only positive values enter (registers start at 0).  Z_i cancels in the L1
// renormalisation, so selection runs on the raw sums.
// Optional by-product: the entropy of the
// Gaussian's aggregated coefficient distribution before Top-K, w_l = W_l / sum W (Z cancels),
// H = -sum_l w_l ln w_l = ln S - (sum_l W_l ln W_l) / S with S = sum_l W_l, accumulated in the
// same pass (fp32; NaN for an empty row).
// Rows are staged through shared memory: the CTA's 128 consecutive rows (128 L floats,
// contiguous in W) are read with coalesced float4 loads -- summed over the P partials in rank
// order 0..P-1 for the fused cross-rank path (peers.n > 1) -- into padded shared rows (stride
// L + 4 floats: a warp's LDS.128 of one column hits 8 distinct 16-B bank groups per wavefront),
// then each thread runs the register insertion network on its own row.
// Shift-insert of atom a (value v) into the list of the KMAX best so far, ordered (value desc,
// atom asc).  Atoms arrive in ascending order, so v goes after every equal value (strict >):
// the entries from its position on shift down by one and the last drops out.  (Comparing the
// displaced entries again instead, as a bubble would, can drop an earlier atom of a tied value.)
template <int KMAX>
__device__ __forceinline__ void topk_insert(float (&bv)[KMAX], uint32_t (&ba)[KMAX], float v, uint32_t a) {
    float nv[KMAX];
    uint32_t na[KMAX];
#pragma unroll
    for (int s = 0; s < KMAX; s++) {
        const bool here = v > bv[s];                    // v goes at or above slot s
        const bool above = s > 0 && v > bv[s - 1];      // ... strictly above: slot s takes s - 1
        nv[s] = above ? bv[s - 1] : (here ? v : bv[s]);
        na[s] = above ? ba[s - 1] : (here ? a : ba[s]);
    }
#pragma unroll
    for (int s = 0; s < KMAX; s++) {
        bv[s] = nv[s];
        ba[s] = na[s];
    }
}

// The 8th largest of 16 values: both halves sorted descending (the optimal 19-comparator network
// for 8), then the top 8 of the union are max(a_i, b_(7-i)) and their minimum is the 8th largest.
__device__ __forceinline__ float eighth_of_16(float (&m)[16]) {
    constexpr int net[19][2] = {{0, 2}, {1, 3}, {4, 6}, {5, 7}, {0, 4}, {1, 5}, {2, 6}, {3, 7}, {0, 1}, {2, 3},
                                {4, 5}, {6, 7}, {2, 4}, {3, 5}, {1, 4}, {3, 6}, {1, 2}, {3, 4}, {5, 6}};
#pragma unroll
    for (int h = 0; h < 16; h += 8)
#pragma unroll
        for (int k = 0; k < 19; k++) {
            const float a = m[h + net[k][0]], b = m[h + net[k][1]];
            m[h + net[k][0]] = fmaxf(a, b);
            m[h + net[k][1]] = fminf(a, b);
        }
    float t = fmaxf(m[0], m[15]);
#pragma unroll
    for (int i = 1; i < 8; i++) t = fminf(t, fmaxf(m[i], m[15 - i]));
    return t;
}

// bit 4 (c4 - ca) + u: value u of float4 column c4 in [ca, cb) is >= tp
__device__ __forceinline__ uint32_t candidate_bits(const float4* row, int ca, int cb, float tp) {
    // set.ge gives an all-ones / zero word per value; each bit is one AND-OR (LOP3) into the mask
    auto ge = [](float v, float t) {
        uint32_t r;
        asm("set.ge.u32.f32 %0, %1, %2;" : "=r"(r) : "f"(v), "f"(t));
        return r;
    };
    uint32_t m = 0u;
    for (int c4 = ca; c4 < cb; c4++) {
        const float4 v4 = row[c4];
        const int sh = 4 * (c4 - ca);
        m |= ge(v4.x, tp) & (1u << sh);
        m |= ge(v4.y, tp) & (2u << sh);
        m |= ge(v4.z, tp) & (4u << sh);
        m |= ge(v4.w, tp) & (8u << sh);
    }
    return m;
}

#ifndef SCOUP_TOPK_ROWS
#define SCOUP_TOPK_ROWS 128
#endif
constexpr int TOPK_ROWS = SCOUP_TOPK_ROWS;

// LC: L / 4 at compile time (the common L = 64: constant row offsets and bit positions), or 0
template <int KMAX, int LC>
__global__ void __launch_bounds__(TOPK_ROWS) topk_tile_kernel(PeerRows peers, int64_t rows, int64_t valid_rows, int L,
                                                              int K, uint32_t* __restrict__ atoms,
                                                              float* __restrict__ coefs, float* __restrict__ entropy) {
    extern __shared__ __align__(16) float tile[];
    if (LC) L = 4 * LC;
    const int L4 = LC ? LC : (L >> 2), LP = L + 4;
    const int R = blockDim.x;  // rows per tile (one per thread)
    const int64_t r0 = (int64_t)blockIdx.x * R;
    const int64_t left = valid_rows - r0;
    const int nr = left < (int64_t)R ? (int)left : R;  // rows of this tile to read
    const int t = threadIdx.x;
    const int n4 = nr > 0 ? nr * L4 : 0;
    const float4* src0 = reinterpret_cast<const float4*>(peers.W[0]) + r0 * L4;  // contiguous row block
    if (peers.n == 1) {
        // one partial: asynchronous copies straight into the padded rows (every thread's 16-B
        // copies in flight at once), then one wait
        for (int i = t; i < n4; i += R) {
            const int rr = i / L4, c4 = i - rr * L4;
            const uint32_t sa = (uint32_t)__cvta_generic_to_shared(tile + rr * LP + 4 * c4);
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(src0 + i));
        }
        asm volatile("cp.async.commit_group;\n" ::);
        asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    } else {
        // P partials summed in rank order 0..P-1, four float4 columns per thread in flight
        for (int i0 = t; i0 < n4; i0 += 4 * R) {
            float4 v[4];
#pragma unroll
            for (int u = 0; u < 4; u++)
                if (i0 + u * R < n4) v[u] = __ldg(src0 + i0 + u * R);
            for (int q = 1; q < peers.n; q++) {
                const float4* srcq = reinterpret_cast<const float4*>(peers.W[q]) + r0 * L4;
#pragma unroll
                for (int u = 0; u < 4; u++)
                    if (i0 + u * R < n4) {
                        const float4 w4 = __ldg(srcq + i0 + u * R);
                        v[u].x = __fadd_rn(v[u].x, w4.x);
                        v[u].y = __fadd_rn(v[u].y, w4.y);
                        v[u].z = __fadd_rn(v[u].z, w4.z);
                        v[u].w = __fadd_rn(v[u].w, w4.w);
                    }
            }
#pragma unroll
            for (int u = 0; u < 4; u++)
                if (i0 + u * R < n4) {
                    const int i = i0 + u * R, rr = i / L4, c4 = i - rr * L4;
                    *reinterpret_cast<float4*>(tile + rr * LP + 4 * c4) = v[u];
                }
        }
    }
    __syncthreads();
    const int64_t r = r0 + t;
    float bv[KMAX];
    uint32_t ba[KMAX];
    float hs = 0.f, hw = 0.f;  // sum W, sum W ln W
#pragma unroll
    for (int s = 0; s < KMAX; s++) { bv[s] = 0.f; ba[s] = NONE; }
    if (t < nr) {
        const float4* row = reinterpret_cast<const float4*>(tile + t * LP);
        const float* rowf = tile + t * LP;
        if (entropy) {
            for (int c4 = 0; c4 < L4; c4++) {
                const float4 v4 = row[c4];
                const float vals[4] = {v4.x, v4.y, v4.z, v4.w};
#pragma unroll
                for (int u = 0; u < 4; u++)
                    if (vals[u] > 0.f) {
                        hs += vals[u];
                        hw += vals[u] * logf(vals[u]);
                    }
            }
        }
        // Candidate bound: the maxima of K disjoint groups of atoms are K distinct elements, so at
        // least K values are >= their minimum tau and no value below tau is in the Top-K.  Only
        // the positive values >= tau (typically ~L/4 of a dense row) go through the insertion
        // network -- in atom order, so ties keep the lower atom (strict >): the same selection and
        // order as inserting every value.
        float tau = 0.f;
        if (LC == 16 && KMAX == 8) {
            // L = 64, K <= 8: the maxima of the 16 float4 groups are 16 distinct elements, so at
            // least 8 >= K values are >= the 8th largest of them (~the row's 84th percentile for
            // dense rows, against ~73rd for the minimum of K group maxima): fewer candidates
            float m[16];
#pragma unroll
            for (int c4 = 0; c4 < 16; c4++) {
                const float4 v4 = row[c4];
                m[c4] = fmaxf(fmaxf(v4.x, v4.y), fmaxf(v4.z, v4.w));
            }
            tau = eighth_of_16(m);
        } else if (L >= K) {
            const int gs = L / K;
            tau = __int_as_float(0x7f800000);
            if ((gs & 3) == 0) {  // float4 groups (conflict-free LDS.128 on the padded rows)
                const int g4 = gs >> 2;
                for (int g = 0; g < K; g++) {
                    const int c1 = g == K - 1 ? L4 : (g + 1) * g4;
                    float m = 0.f;
                    for (int c4 = g * g4; c4 < c1; c4++) {
                        const float4 v4 = row[c4];
                        m = fmaxf(m, fmaxf(fmaxf(v4.x, v4.y), fmaxf(v4.z, v4.w)));
                    }
                    tau = fminf(tau, m);
                }
            } else {
                for (int g = 0; g < K; g++) {
                    const int a0 = g * gs, a1 = g == K - 1 ? L : a0 + gs;
                    float m = rowf[a0];
                    for (int a = a0 + 1; a < a1; a++) m = fmaxf(m, rowf[a]);
                    tau = fminf(tau, m);
                }
            }
        }
        // candidates: v >= tau and v > 0, i.e. v >= max(tau, the smallest positive float)
        const float tp = fmaxf(tau, __int_as_float(1));
        for (int c0 = 0; c0 < L4; c0 += 16) {  // chunks of 64 atoms: a candidate bit mask each
            const uint32_t lo = candidate_bits(row, c0, min(L4, c0 + 8), tp);  // (two 32-bit halves)
            const uint32_t hi = candidate_bits(row, c0 + 8, min(L4, c0 + 16), tp);
            unsigned long long cm = ((unsigned long long)hi << 32) | lo;
            while (cm) {
                const int bit = __ffsll((long long)cm) - 1;
                cm &= cm - 1ull;
                const uint32_t a = (uint32_t)(4 * c0 + bit);
                const float v = rowf[a];
                if (v > bv[KMAX - 1]) topk_insert<KMAX>(bv, ba, v, a);
            }
        }
    }
    float sum = 0.f;
#pragma unroll
    for (int s = 0; s < KMAX; s++)
        if (s < K) sum = __fadd_rn(sum, bv[s]);
    // w = v / sum as v * (1 / sum): two roundings (<= 1.5 ulp, inside Eq. 6's fp32 tolerance) and
    // monotone in v, so the stored coefficients keep the selection's descending order
    const float inv = __frcp_rn(sum);
    if (entropy && r < rows) entropy[r] = hs > 0.f ? fmaxf(0.f, logf(hs) - hw / hs) : __int_as_float(0x7fc00000);
    if (2 * K > L + 4) {  // (codes wider than half a staged row: direct stores)
        if (r < rows) {
#pragma unroll
            for (int s = 0; s < KMAX; s++) {
                if (s < K) {
                    bool keep = bv[s] > 0.f;
                    atoms[r * K + s] = keep ? ba[s] : NONE;
                    coefs[r * K + s] = keep ? __fmul_rn(bv[s], inv) : 0.f;
                }
            }
        }
        return;
    }
    // the tile's codes through shared memory (every row has been read: the tile is free), then
    // one contiguous, coalesced store of its R x K atoms and coefficients
    __syncthreads();
    uint32_t* oa = reinterpret_cast<uint32_t*>(tile);
    float* oc = tile + R * K;
#pragma unroll
    for (int s = 0; s < KMAX; s++) {
        if (s < K) {
            bool keep = bv[s] > 0.f;
            oa[t * K + s] = keep ? ba[s] : NONE;
            oc[t * K + s] = keep ? __fmul_rn(bv[s], inv) : 0.f;
        }
    }
    __syncthreads();
    const int64_t left_rows = rows - r0;
    const int nout = (int)(left_rows < (int64_t)R ? left_rows : (int64_t)R) * K;
    for (int k = t; k < nout; k += R) {
        atoms[r0 * K + k] = oa[k];
        coefs[r0 * K + k] = oc[k];
    }
}

// generic L (not a multiple of 4): scalar loads
template <int KMAX>
__global__ void __launch_bounds__(128) topk_kernel_scalar(const float* __restrict__ W, int64_t rows,
                                                          int64_t valid_rows, int L, int K,
                                                          uint32_t* __restrict__ atoms, float* __restrict__ coefs,
                                                          float* __restrict__ entropy) {
    int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= rows) return;
    float bv[KMAX];
    uint32_t ba[KMAX];
    float hs = 0.f, hw = 0.f;
#pragma unroll
    for (int s = 0; s < KMAX; s++) { bv[s] = 0.f; ba[s] = NONE; }
    if (r < valid_rows) {
        for (int c = 0; c < L; c++) {
            float v = __ldg(W + r * (int64_t)L + c);
            if (entropy && v > 0.f) {
                hs += v;
                hw += v * logf(v);
            }
            if (v > bv[KMAX - 1]) topk_insert<KMAX>(bv, ba, v, (uint32_t)c);
        }
    }
    float sum = 0.f;
#pragma unroll
    for (int s = 0; s < KMAX; s++)
        if (s < K) sum = __fadd_rn(sum, bv[s]);
    // w = v / sum as v * (1 / sum): two roundings (<= 1.5 ulp, inside Eq. 6's fp32 tolerance) and
    // monotone in v, so the stored coefficients keep the selection's descending order
    const float inv = __frcp_rn(sum);
#pragma unroll
    for (int s = 0; s < KMAX; s++) {
        if (s < K) {
            bool keep = bv[s] > 0.f;
            atoms[r * K + s] = keep ? ba[s] : NONE;
            coefs[r * K + s] = keep ? __fdiv_rn(bv[s], sum) : 0.f;
        }
    }
    if (entropy) entropy[r] = hs > 0.f ? fmaxf(0.f, logf(hs) - hw / hs) : __int_as_float(0x7fc00000);
}

}  // namespace

int select_tiles_per_view(int64_t G) { return (int)grid_for(G, SEL_TILE); }

size_t select_counts_needed(int64_t G, int nviews) {
    return (size_t)grid_for(G, SEL_TILE) * (size_t)nviews * (1 + 8 * SEL_ITEMS);
}

void launch_select_far2(const ViewBuffers& vb, PackedGaussians pg, int64_t G, int nviews, int key_bits,
                        const Binning& bn, uint32_t* counts, cudaStream_t s) {
    if (G <= 0 || nviews <= 0) return;
    uint16_t* sat = reinterpret_cast<uint16_t*>(vb.live_sat);
    live_sat_kernel<<<nviews, 1024, 0, s>>>(vb.tile_live, bn.tiles_x, bn.tiles_y, sat);
    const bool packed = bn.tiles_x <= 255 && bn.tiles_y <= 255;
    const FarSel pred{vb.code, vb.thr, G, (1u << key_bits) - 1u, packed ? vb.trect : nullptr, sat,
                      bn.tiles_x, bn.tiles_y, pg, vb.cams};
    compact(pred, G, nviews, counts, vb.sel, vb.nsel, s);
}

void launch_activate(const float* means, const float* scales, const float* rots, const float* opac, int64_t G,
                     PackedGaussians pg, ErrorLatch err, cudaStream_t s) {
    if (G <= 0) return;
    activate_kernel<<<grid_for(G, 256), 256, 0, s>>>(means, scales, rots, opac, G, pg, err);
}

void launch_bounds(PackedGaussians pg, int64_t G, int* bbox, cudaStream_t s) {
    if (G <= 0) return;
    const int64_t blocks = std::min<int64_t>((G + 255) / 256, 1184);
    bounds_kernel<<<(unsigned)blocks, 256, 0, s>>>(pg, G, bbox);
}

void launch_depth_hist(PackedGaussians pg, int64_t G, const CamBatch& cams, int key_bits, uint32_t* hist,
                       cudaStream_t s) {
    if (G <= 0 || cams.n <= 0) return;
    const int64_t n = (G + HIST_SAMPLE - 1) / HIST_SAMPLE;
    dim3 grid((unsigned)std::min<int64_t>((n + 255) / 256, 64), (unsigned)cams.n);
    depth_hist_kernel<<<grid, 256, 0, s>>>(pg, G, cams, key_bits, hist);
}

void launch_depth_pass_near(PackedGaussians pg, int64_t G, const CamBatch& cams, int key_bits, const uint32_t* thr,
                            uint32_t* code, unsigned long long* visible_ctr, ErrorLatch err, const Binning& bn,
                            uint32_t* trect, uint32_t* counts, uint32_t* sel, int* nsel, cudaStream_t s) {
    if (G <= 0 || cams.n <= 0) return;
    const dim3 grid(grid_for(G, SEL_TILE), (unsigned)cams.n);
    const int64_t tiles = (int64_t)grid.x * grid.y;
    uint32_t* bits = counts + tiles;
    const bool packed = bn.tiles_x <= 255 && bn.tiles_y <= 255;
    depth_pass_kernel<<<grid.x, 256, 0, s>>>(pg, G, cams, key_bits, thr, code, visible_ctr, err, bn.tiles_x, bn.tiles_y,
                                             packed ? trect : nullptr, counts, bits);
    sel_scan_kernel<<<1, 1024, 0, s>>>(counts, (int)tiles, nsel);
    sel_scatter_kernel<<<grid, 256, 0, s>>>(G, counts, bits, sel);
}

void launch_preprocess(PackedGaussians pg, int64_t G, const CamBatch& cams, Binning bn, ViewBuffers vb,
                       int key_bits, int64_t nsel, cudaStream_t s) {
    if (nsel <= 0) return;
    preprocess_kernel<<<grid_for(nsel, 256), 256, 0, s>>>(pg, G, cams, bn, vb, key_bits, vb.sel, nsel, vb.skey,
                                                          vb.sval);
}

void launch_ingest_dense(const float* in, int64_t n, float* out, ErrorLatch err, cudaStream_t s) {
    if (n <= 0) return;
    ingest_dense_kernel<<<grid_for(n, 256), 256, 0, s>>>(in, n, out, err);
}

void launch_ingest_codes(const uint32_t* atoms_in, const float* coefs_in, int64_t rows, int S, int K, int L,
                         uint32_t* atoms_out, float* coefs_out, ErrorLatch err, cudaStream_t s) {
    if (rows <= 0) return;
    ingest_codes_kernel<<<grid_for(rows, 128), 128, 0, s>>>(atoms_in, coefs_in, rows, S, K, L, atoms_out,
                                                            coefs_out, err);
}

// Fused cross-rank reduction + Top-K (SURVEY.md §8(e)'s fusion option): the rows of this rank's
// shard are summed over the P ranks' partial accumulators in place -- read directly from the
// peers' memory (CUDA IPC mappings over NVLink / NVSwitch), in rank order 0..P-1 -- and Eq. 6
// runs on the sums (topk_tile_kernel with P partials).  This replaces reduce-scatter + Top-K: no
// reduced shard is written and re-read.
template <int KMAX, int LC>
static void topk_tile_launch(PeerRows peers, int64_t rows, int64_t valid_rows, int L, int K, uint32_t* atoms,
                             float* coefs, float* entropy, cudaStream_t s) {
    const int R = L <= 256 ? TOPK_ROWS : 32;  // rows per CTA: <= 133 KB of staged rows (L <= SCOUP_MAX_L)
    const size_t smem = (size_t)R * (L + 4) * sizeof(float);
    static int smem_set = 0;  // opt-in above 48 KB, once per instantiation and size
    if (smem > 48 * 1024 && smem_set < (int)smem) {
        cudaFuncSetAttribute(topk_tile_kernel<KMAX, LC>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        smem_set = (int)smem;
    }
    topk_tile_kernel<KMAX, LC><<<grid_for(rows, R), R, smem, s>>>(peers, rows, valid_rows, L, K, atoms, coefs, entropy);
}

template <int KMAX>
static void topk_tile_l(PeerRows peers, int64_t rows, int64_t valid_rows, int L, int K, uint32_t* atoms,
                        float* coefs, float* entropy, cudaStream_t s) {
    if (L == 64) topk_tile_launch<KMAX, 16>(peers, rows, valid_rows, L, K, atoms, coefs, entropy, s);
    else topk_tile_launch<KMAX, 0>(peers, rows, valid_rows, L, K, atoms, coefs, entropy, s);
}

static void topk_tile(const PeerRows& peers, int64_t rows, int64_t valid_rows, int L, int K, uint32_t* atoms,
                      float* coefs, float* entropy, cudaStream_t s) {
    if (K <= 4) topk_tile_l<4>(peers, rows, valid_rows, L, K, atoms, coefs, entropy, s);
    else if (K <= 8) topk_tile_l<8>(peers, rows, valid_rows, L, K, atoms, coefs, entropy, s);
    else if (K <= 16) topk_tile_l<16>(peers, rows, valid_rows, L, K, atoms, coefs, entropy, s);
    else topk_tile_l<32>(peers, rows, valid_rows, L, K, atoms, coefs, entropy, s);
}

void launch_topk_peers(const PeerRows& peers, int64_t first_row, int64_t rows, int64_t valid_rows, int L, int K,
                       uint32_t* atoms, float* coefs, cudaStream_t s) {
    if (rows <= 0) return;
    PeerRows pr = peers;
    for (int q = 0; q < pr.n; q++) pr.W[q] = peers.W[q] + first_row * (int64_t)L;
    topk_tile(pr, rows, valid_rows, L, K, atoms, coefs, nullptr, s);  // (the caller checked L % 4, alignment)
}

template <int KMAX>
static void topk_dispatch_scalar(const float* W, int64_t rows, int64_t valid_rows, int L, int K, uint32_t* atoms,
                                 float* coefs, float* entropy, cudaStream_t s) {
    topk_kernel_scalar<KMAX><<<grid_for(rows, 128), 128, 0, s>>>(W, rows, valid_rows, L, K, atoms, coefs, entropy);
}

void launch_topk(const float* W, int64_t rows, int64_t valid_rows, int L, int K, uint32_t* atoms, float* coefs,
                 float* entropy, cudaStream_t s) {
    if (rows <= 0) return;
    if (L % 4 == 0 && (reinterpret_cast<uintptr_t>(W) % 16) == 0) {
        PeerRows pr{};
        pr.W[0] = W;
        pr.n = 1;
        topk_tile(pr, rows, valid_rows, L, K, atoms, coefs, entropy, s);
        return;
    }
    if (K <= 4) topk_dispatch_scalar<4>(W, rows, valid_rows, L, K, atoms, coefs, entropy, s);
    else if (K <= 8) topk_dispatch_scalar<8>(W, rows, valid_rows, L, K, atoms, coefs, entropy, s);
    else if (K <= 16) topk_dispatch_scalar<16>(W, rows, valid_rows, L, K, atoms, coefs, entropy, s);
    else topk_dispatch_scalar<32>(W, rows, valid_rows, L, K, atoms, coefs, entropy, s);
}

}  // namespace scoup
