// internal.cuh -- shared declarations of the sm_100a CUDA path (not part of the C ABI).
//
// Parity-critical arithmetic is written with explicit round-to-nearest
// intrinsics (__fmul_rn, __fadd_rn, __fdiv_rn, __fsqrt_rn, __fmaf_rn) so that no
// compiler contraction or fast-math flag can change a rounding; the TU is also built
// with -fmad=false.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace scoup {

constexpr uint32_t NONE = 0xFFFFFFFFu;
constexpr int TILE = 16;                 // 16x16 pixel tiles, one CTA (256 threads) each
constexpr int TILE_PIX = TILE * TILE;
constexpr int BATCH = 32;                // Gaussians staged per raster batch
constexpr int MAX_SLOTS = 32;            // distinct regions per tile on the smem-aggregated path
constexpr int MAX_S = 16;
constexpr int MAX_VB = 8;                // views batched per preprocess/sort/raster pass
constexpr int MAX_BINS = 2048;           // bins per view batch (views x bins per view)

// DESIGN.md §3 constants (hex-exact fp32)
#define K_NEAR 0x1.99999ap-3f
#define K_LOWPASS 0x1.333334p-2f
#define K_ACLAMP 0x1.fae148p-1f
#define K_AMIN 0x1.010102p-8f
#define K_TMIN 0x1.a36e2ep-14f
#define K_HALF_LOG2E (-0x1.715476p-1f)
#define K_LOG2E_NEG (-0x1.715476p+0f)

// Pixel tiling: 16x16 raster tiles, grouped into power-of-two bins (multiples of a tile) whose
// depth-ordered Gaussian lists are what the binning sort produces.
struct Binning {
    int tiles_x, tiles_y;   // raster tiles
    int bshx, bshy;         // log2 of the bin size in pixels (>= 4)
    int bins_x, bins_y;     // bins
    __host__ __device__ int nbins() const { return bins_x * bins_y; }
};

struct Camera {
    float fx, fy, cx, cy;
    int width, height;
    float P[12];  // rows of [R|t]
};

// Packed, activated Gaussians (derived once in init, DESIGN.md §3 G1).
struct PackedGaussians {
    float4* a;   // (mx, my, mz, o)   o < 0 marks an invalid Gaussian
    float4* b;   // (V00, V01, V02, V11)
    float2* c;   // (V12, V22)
};

// A batch of B <= MAX_VB views is projected, sorted and rasterised together.  Per-view,
// per-Gaussian arrays are [B*G], indexed by the batch index j = v*G + i (view v, Gaussian i).
//   rec0 = (mean2d.x, mean2d.y, r, o)     rec1 = (qa, qb, qc, ycut)
struct ViewBuffers {
    uint32_t* depth_key;     // [B*G] (v << nb) | depth code (DESIGN.md §5 a3), invisible: all ones
    uint32_t* depth_key_alt; // [B*G] sort scratch
    uint32_t* dval;          // [B*G] batch index j (iota)
    uint32_t* dval_sorted;   // [B*G] batch indices in (view, depth, index) order
    uint32_t* tiles;         // [B*G] bin count of the support rectangle
    uint64_t* offsets;       // [B*G] inclusive scan of tiles in sorted order
    uint2* rect;             // [B*G] bin rect (bx0 | by0<<16, bx1 | by1<<16), exclusive ends
    float4* rec0;            // [B*G]
    float4* rec1;            // [B*G]
    float2* rec2;            // [B*G] half-extents of the conservative support box (GPU-only prune)
    uint64_t* totals;        // [MAX_VB] offsets at the end of each view
    uint32_t* ekey;          // [E] v*nbins + bin of each (Gaussian, bin) entry
    uint32_t* eval;          // [E] batch index j
    uint32_t* ekey_alt;      // [E] sort scratch
    uint32_t* eval_alt;      // [E]
    uint2* ranges;           // [B*nbins] [begin, end) into the sorted entries
    uint32_t* bin_count;     // [B*nbins] entries per bin (histogram of emission)
};

struct CamBatch {
    Camera cam[MAX_VB];
    int n;                   // views in the batch
};

struct ErrorLatch {
    int* code;         // device: 0 = none, else SCOUP_EDATA kind id
    long long* index;  // device: first offending index
};

enum DataErr : int { ERR_NONE = 0, ERR_GAUSSIAN = 1, ERR_REGION = 2, ERR_CODE = 3, ERR_DEPTHKEY = 4 };

__device__ __forceinline__ void latch_error(ErrorLatch e, int kind, long long idx) {
    if (atomicCAS(e.code, 0, kind) == 0) *e.index = idx;
}

// ---- launchers (kernels.cu) ----
void launch_activate(const float* means, const float* scales, const float* rots, const float* opac,
                     int64_t G, PackedGaussians pg, ErrorLatch err, cudaStream_t s);
void launch_bounds(PackedGaussians pg, int64_t G, int* bbox, cudaStream_t s);
void launch_preprocess(PackedGaussians pg, int64_t G, const CamBatch& cams, Binning bn, ViewBuffers vb,
                       int key_bits, unsigned long long* visible_ctr, ErrorLatch err, cudaStream_t s);
void launch_gather_scan_input(const uint32_t* dval_sorted, const uint32_t* tiles, uint64_t* out,
                              int64_t n, cudaStream_t s);
void launch_view_totals(const uint64_t* offsets, int64_t G, int nviews, uint64_t* totals, cudaStream_t s);
void launch_emit(const uint32_t* dval_sorted, const uint64_t* offsets, const uint2* rect, Binning bn,
                 int64_t n, int64_t G, uint32_t* ekey, uint32_t* eval, uint32_t* bin_count, cudaStream_t s);
void launch_ranges_from_counts(const uint32_t* bin_count, int nbins, uint2* ranges, cudaStream_t s);
void launch_ingest_codes(const uint32_t* atoms_in, const float* coefs_in, int64_t rows, int S, int K,
                         int L, uint32_t* atoms_out, float* coefs_out, ErrorLatch err, cudaStream_t s);

struct RasterParams {
    int nviews;                   // views in the batch; grid = nviews x tiles
    int width, height;
    int64_t G;                    // Gaussians (batch index j = v*G + i)
    Binning bn;
    const uint2* ranges;          // [nviews * nbins]
    const uint32_t* eval;         // sorted entries: batch indices
    const float4* rec0;           // [nviews * G]
    const float4* rec1;
    const float2* rec2;
    const uint32_t* region_ids[MAX_VB];  // [H*W] per view
    int64_t code_row0[MAX_VB];
    int32_t num_regions[MAX_VB];
    long long pixel_base[MAX_VB];        // flat index of the view's first pixel (error reports)
    long long* contrib_out[MAX_VB];      // optional per-view counters
    const uint32_t* code_atoms;   // sanitised table, rows of S slots
    const float* code_coefs;
    int S;
    int L;
    float* W;
    float* Z;
    unsigned long long* contrib_ctr;  // handle stats
    unsigned long long* support_ctr;  // handle stats: support tests
    ErrorLatch err;
};
void launch_raster(const RasterParams& p, cudaStream_t s);

void launch_topk(const float* W, int64_t rows, int64_t valid_rows, int L, int K, uint32_t* atoms,
                 float* coefs, cudaStream_t s);

}  // namespace scoup
