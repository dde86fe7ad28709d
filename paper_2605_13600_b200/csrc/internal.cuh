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
constexpr int MAX_SAT_ENTRIES = 12288;   // (tiles_x + 1) * (tiles_y + 1): 1920x1080 needs 121 x 69
constexpr int HIST_BITS = 10;            // depth-code histogram resolution (near/far split)
constexpr int NHIST = 1 << HIST_BITS;

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
    float* s2;   // max(s)^2 (slightly padded): conservative reach of the chunk predicates
};

struct CamBatch {
    Camera cam[MAX_VB];
    int n;                   // views in the batch
};

// A batch of B <= MAX_VB views is processed together, in two depth chunks (DESIGN.md §5 a3):
// per-(view, Gaussian) arrays are [B*G], indexed by the batch index j = v*G + i.
//   rec0 = (mean2d.x, mean2d.y, r, o)     rec1 = (qa, qb, qc, ycut)     rec2 = (box ext x, y, id, 0)
struct ViewBuffers {
    uint32_t* code;          // [B*G] depth code (bits(t_z) - bits(0.2f)), all ones = invisible
    uint32_t* hist;          // [B*NHIST] histogram of the codes' top bits, per view
    uint32_t* thr;           // [MAX_VB] near/far split code per view
    CamBatch* cams;          // device copy of the batch's cameras (chunk predicates)
    uint32_t* sel;           // [B*G] batch indices selected for the current chunk (index order)
    int* nsel;               // device count of sel
    uint32_t* skey;          // [B*G] (v << key_bits) | code of the selected elements
    uint32_t* skey_alt;      // [B*G] sort scratch
    uint32_t* sval;          // [B*G] chunk index e (position in sel)
    uint32_t* sval_sorted;   // [B*G] chunk indices in (view, depth, index) order
    // per selected element e of the current chunk (compact, written in sel order):
    uint32_t* tiles;         // bin count of the support rectangle
    uint64_t* offsets;       // [B*G] inclusive scan of tiles in sorted order
    uint2* rect;             // bin rect (bx0 | by0<<16, bx1 | by1<<16), exclusive ends
    float4* rec0;
    float4* rec1;
    float4* rec2;            // (support box half-extents x, y, Gaussian id bits, 0)
    float* Tstate;           // [B*H*W] per-pixel transmittance between chunks (0 = finished)
    uint8_t* tile_live;      // [B*tiles] 1 while a tile has an unfinished pixel
    uint8_t* flags;          // [B*G] far-chunk selection flags
    uint32_t* live_sat;      // [B*(tiles_x+1)*(tiles_y+1)] summed-area table of tile_live
    uint32_t* ekey;          // [E] v*nbins + bin of each (Gaussian, bin) entry
    uint32_t* eval;          // [E] batch index j
    uint32_t* ekey_alt;      // [E] sort scratch
    uint32_t* eval_alt;      // [E]
    uint2* ranges;           // [B*nbins] [begin, end) into the sorted entries
    uint32_t* bin_count;     // [B*nbins] entries per bin (histogram of emission)
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
void launch_depth_pass(PackedGaussians pg, int64_t G, const CamBatch& cams, int key_bits, uint32_t* code,
                       uint32_t* hist, unsigned long long* visible_ctr, ErrorLatch err, cudaStream_t s);
// stable compactions into vb.sel / vb.nsel; temp storage grown through *tmp / *tmp_bytes
size_t select_temp_bytes(int64_t n);
void launch_select_near(const ViewBuffers& vb, int64_t G, int nviews, int key_bits, void* tmp, size_t tmp_bytes,
                        cudaStream_t s);
void launch_select_flagged(const ViewBuffers& vb, const uint8_t* flags, int64_t n, void* tmp, size_t tmp_bytes,
                           cudaStream_t s);
void launch_preprocess(PackedGaussians pg, int64_t G, const CamBatch& cams, Binning bn, ViewBuffers vb,
                       int key_bits, int64_t nsel, cudaStream_t s);
void launch_gather_scan_input(const uint32_t* sval_sorted, const uint32_t* tiles, uint64_t* out, int64_t n,
                              cudaStream_t s);
void launch_emit(const uint32_t* sval_sorted, const uint32_t* skey_sorted, int key_bits, const uint64_t* offsets,
                 const uint2* rect, Binning bn, int64_t n, int nviews, uint32_t* ekey, uint32_t* eval,
                 uint32_t* bin_count, cudaStream_t s);
void launch_far_flags(const ViewBuffers& vb, PackedGaussians pg, int64_t G, const CamBatch& cams, int key_bits,
                      const Binning& bn, uint8_t* flags, cudaStream_t s);
void launch_ranges_from_counts(const uint32_t* bin_count, int nbins, uint2* ranges, cudaStream_t s);
void launch_ingest_codes(const uint32_t* atoms_in, const float* coefs_in, int64_t rows, int S, int K,
                         int L, uint32_t* atoms_out, float* coefs_out, ErrorLatch err, cudaStream_t s);

struct RasterParams {
    int nviews;                   // views in the batch; grid = nviews x tiles
    int width, height;
    int64_t G;                    // Gaussians (batch index j = v*G + i)
    Binning bn;
    const uint2* ranges;          // [nviews * nbins]
    const uint32_t* eval;         // sorted entries: chunk indices e
    const float4* rec0;           // [nviews * G]
    const float4* rec1;
    const float4* rec2;
    float* Tstate;                // [nviews * H*W] transmittance carried between chunks
    uint8_t* tile_live;           // [nviews * tiles]
    int chunk;                    // 0: first chunk (T starts at 1), else continue from Tstate
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
