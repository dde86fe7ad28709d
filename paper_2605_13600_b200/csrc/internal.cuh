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
constexpr int MAX_SLOTS = 16;            // distinct region(-tuple)s per tile on the smem-aggregated path
constexpr int MAX_S = 16;
#ifndef SCOUP_MAX_VB
#define SCOUP_MAX_VB 16
#endif
constexpr int MAX_VB = SCOUP_MAX_VB;     // views batched per preprocess/sort/raster pass
constexpr int MAX_LEV = 4;               // semantic levels fused per raster pass (nlev * S <= MAX_S)
constexpr int MAX_SAT_ENTRIES = 12288;   // (tiles_x + 1) * (tiles_y + 1): 1920x1080 needs 121 x 69
constexpr int HIST_BITS = 10;            // depth-code histogram resolution (near/far split)
constexpr int NHIST = 1 << HIST_BITS;
constexpr int HIST_SAMPLE = 32;          // the depth histogram counts every 32nd Gaussian

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
//   rec0 = (mean2d.x, mean2d.y, r, o)     rec1 = (qa, qb, qc, ycut)
//   rec2 = (box ext x, y, id, sy)         rec3 = span parameters (band_relevant)
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
    uint2* rect;             // bin rect (bx0 | by0<<16, bx1 | by1<<16), exclusive ends
    float4* rec0;
    float4* rec1;
    float4* rec2;            // (support box half-extents x, y, Gaussian id bits, sy)
    float4* rec3;            // (ky/(-qa), yc/(-qa), -qb/(2 qa), sx): band_relevant parameters
    float* Tstate;           // [B*H*W] per-pixel transmittance between chunks (0 = finished)
    uint8_t* tile_live;      // [B*tiles] 1 while a tile has an unfinished pixel
    uint32_t* selcnt;        // tile counts / offsets of the stable compactions
    uint32_t* trect;         // [B*G] conservative reach box in 16x16 tiles (x0, x1, y0, y1: 8 bits each),
                             //       written by the depth pass for the far-chunk predicate
    uint32_t* live_sat;      // [B*(tiles_x+1)*(tiles_y+1)] summed-area table of tile_live
    uint32_t* eval;          // [E] chunk element index of each (bin, element) entry, bin lists in depth order
    uint2* ranges;           // [B*nbins] [begin, end) of each bin's list in eval
    uint32_t* bcnt;          // [segments * nbins] per-segment bin counts / prefixes (binsort.cu)
    uint16_t* ebin;          // [E] bin (within the view) of each flattened entry (binsort.cu)
    uint32_t* eel;           // [E] element of each flattened entry (binsort.cu)
    struct BsInfo* binfo;    // view starts and segment table of the chunk (binsort.cu)
};


// Segment table of the stable bin scatter (binsort.cu): view v's sorted elements are
// [vstart[v], vstart[v+1]) and its flattened entries [ebase[v], ebase[v+1]), cut into runs of
// sege (>= BS_SEGE) entries starting at segment segbase[v].
constexpr int BS_SEGE = 2048;
struct BsInfo {
    uint32_t vstart[MAX_VB + 1];
    uint32_t ebase[MAX_VB + 1];
    uint32_t segbase[MAX_VB + 1];
    uint32_t sege;             // entries per segment (binsort_segment_len)
    unsigned long long total;  // entries of the chunk (exact)
};

struct ErrorLatch {
    int* code;         // device: 0 = none, else SCOUP_EDATA kind id
    long long* index;  // device: first offending index
};

enum DataErr : int { ERR_NONE = 0, ERR_GAUSSIAN = 1, ERR_REGION = 2, ERR_CODE = 3, ERR_DEPTHKEY = 4 };

__device__ __forceinline__ void latch_error(ErrorLatch e, int kind, long long idx) {
    if (atomicCAS(e.code, 0, kind) == 0) *e.index = idx;
}

// Conservative test: may Gaussian (rec0 = mx, my, r, o; rec1 = qa, qb, qc, ycut; ext = support
// box half-extents) produce a
// fragment at a pixel centre inside [X0, X1] x [Y0, Y1]?  A fragment needs |d| <= r (square
// support) and q(d) >= ycut (alpha >= 1/255, ycut already conservative).  Margins make every
// rounding here (and in the pixel's own fp32 evaluation of q, whose absolute error grows with
// the size of the quadratic terms, e.g. for far off-screen near-plane Gaussians) only accept
// more: the rectangle is widened by 0.5 px and ycut relaxed by 0.01 + 2e-6 * (bound on the
// terms of q over the rectangle).  Chords use the Schur form (peak of q along a line,
// 4 qa qc - qb^2 in fp64) so elongated ellipses do not lose precision.
__device__ __forceinline__ bool rect_relevant(float4 a, float4 b, float2 ext, float X0, float X1, float Y0, float Y1) {
    const float mx = a.x, my = a.y, r = a.z;
    // support box of preprocess (square support intersected with the alpha >= 1/255 ellipse's
    // box, padded by >= 1 px): pixel centres outside it never produce a fragment
    if (mx + ext.x < X0 || mx - ext.x > X1 || my + ext.y < Y0 || my - ext.y > Y1) return false;
    const float M = 0.5f;
    X0 -= M; X1 += M; Y0 -= M; Y1 += M;
    // ellipse {q >= yc}: centre inside, or it meets an edge of the rectangle
    if (mx >= X0 && mx <= X1 && my >= Y0 && my <= Y1) return true;
    const float qa = b.x, qb = b.y, qc = b.z;
    const float ex0 = X0 - mx, ex1 = X1 - mx, ey0 = Y0 - my, ey1 = Y1 - my;
    const float dxm = fminf(fmaxf(fabsf(ex0), fabsf(ex1)), r), dym = fminf(fmaxf(fabsf(ey0), fabsf(ey1)), r);
    const float mq = (fabsf(qa) + 0.5f * fabsf(qb)) * dxm * dxm + (fabsf(qc) + 0.5f * fabsf(qb)) * dym * dym;
    const float yc = b.w - 0.01f - 2e-6f * mq;
    const float dq = (float)(4.0 * (double)qa * (double)qc - (double)qb * (double)qb);
    if (!(dq > 0.f)) return true;  // degenerate form: accept
    const float ky = dq / (4.f * qa), kx = dq / (4.f * qc);  // peak of q along a row / column, per d^2
    // rows y = const: q(dx) = qa (dx - c)^2 + ky dy^2 with c = -qb dy / (2 qa)
#pragma unroll
    for (int k = 0; k < 2; k++) {
        const float ey = k ? ey1 : ey0;
        const float h2 = (ky * ey * ey - yc) / -qa;
        if (h2 >= 0.f) {
            const float c = -qb * ey / (2.f * qa), h = sqrtf(h2);
            if (c + h >= ex0 && c - h <= ex1) return true;
        }
    }
#pragma unroll
    for (int k = 0; k < 2; k++) {
        const float ex = k ? ex1 : ex0;
        const float h2 = (kx * ex * ex - yc) / -qc;
        if (h2 >= 0.f) {
            const float c = -qb * ex / (2.f * qc), h = sqrtf(h2);
            if (c + h >= ey0 && c - h <= ey1) return true;
        }
    }
    return false;
}

// Tile-row spans of a Gaussian's possible fragments (GPU-only binning, DESIGN.md §5 a3).  For the
// 16x16 tile row ty, row_span returns the tile columns [tx0, tx1] whose pixel centres may hold
// a fragment: pixel centres inside the support box and inside the alpha >= 1/255 ellipse
// {q >= yc} (yc relaxed as in rect_relevant, with the bound on q's terms taken over the whole
// square support, so it is at least as loose).  Over the row's band (widened by 0.5 px) the
// ellipse's x-extent is at its extreme points (+-sx, +-sy) when they lie in the band, else at
// the band edge nearest to them (the right/left boundary is concave/convex in dy).  The same
// function counts the entries (preprocess) and writes them (emit), so both agree exactly.
struct Span {
    float mx, my, bx, by;   // mean2d, support-box half-extents
    float yc, ky, ia, cq;   // relaxed level, row-peak factor, 1/(-qa), -qb/(2 qa)
    float sx, sy;           // rightmost point of the ellipse relative to the mean (leftmost: -sx, -sy)
    bool box_only;          // degenerate form: use the box
};

__device__ __forceinline__ Span span_setup(float4 a, float4 b, float2 ext) {
    Span s;
    s.mx = a.x; s.my = a.y; s.bx = ext.x; s.by = ext.y;
    const float r = a.z, qa = b.x, qb = b.y, qc = b.z;
    const float mq = ((fabsf(qa) + fabsf(qc)) + fabsf(qb)) * r * r;
    s.yc = b.w - 0.01f - 2e-6f * mq;
    const double dq = 4.0 * (double)qa * (double)qc - (double)qb * (double)qb;
    s.box_only = !(dq > 0.0) || !(qa < 0.f) || !(qc < 0.f) || !(s.yc < 0.f);
    s.ky = (float)(dq / (4.0 * (double)qa));
    s.ia = 1.0f / -qa;
    s.cq = (float)(-(double)qb / (2.0 * (double)qa));
    const double sxd = s.box_only ? 0.0 : sqrt(4.0 * (double)s.yc * (double)qc / dq);
    s.sx = (float)sxd;
    s.sy = s.box_only ? 0.f : (float)(-(double)qb / (2.0 * (double)qc) * sxd);
    return s;
}

__device__ __forceinline__ void row_span(const Span& s, int ty, int tiles_x, int width, int height, int& tx0, int& tx1) {
    tx0 = 1; tx1 = 0;  // empty
    const float Y0 = (float)(ty * TILE) + 0.5f, Y1 = (float)(min(ty * TILE + TILE, height) - 1) + 0.5f;
    if (s.my + s.by < Y0 || s.my - s.by > Y1) return;
    float xl = s.mx - s.bx, xr = s.mx + s.bx;
    if (!s.box_only) {
        const float ey0 = Y0 - 0.5f - s.my, ey1 = Y1 + 0.5f - s.my;
        float rr, ll;
        if (s.sy >= ey0 && s.sy <= ey1) {
            rr = s.sx;
        } else {
            const float ey = s.sy < ey0 ? ey0 : ey1;
            const float h2 = (s.ky * ey * ey - s.yc) * s.ia;
            if (h2 < 0.f) return;  // the band misses the (relaxed) ellipse
            rr = s.cq * ey + sqrtf(h2);
        }
        if (-s.sy >= ey0 && -s.sy <= ey1) {
            ll = -s.sx;
        } else {
            const float ey = -s.sy < ey0 ? ey0 : ey1;
            const float h2 = (s.ky * ey * ey - s.yc) * s.ia;
            if (h2 < 0.f) return;
            ll = s.cq * ey - sqrtf(h2);
        }
        // outward margins: 0.5 px (as rect_relevant) + fp32 rounding of the terms above
        const float mr = 0.5f + 1e-4f * (fabsf(rr) + fabsf(s.mx)) + 1e-3f;
        const float ml = 0.5f + 1e-4f * (fabsf(ll) + fabsf(s.mx)) + 1e-3f;
        xr = fminf(xr, s.mx + rr + mr);
        xl = fmaxf(xl, s.mx + ll - ml);
    }
    if (!(xl <= xr)) return;
    // pixels x whose centre x + 0.5 lies in [xl, xr]
    const float fx0 = fmaxf(ceilf(xl - 0.5f), 0.f), fx1 = fminf(floorf(xr - 0.5f), (float)(width - 1));
    if (!(fx0 <= fx1)) return;
    tx0 = (int)fx0 >> 4;
    tx1 = (int)fx1 >> 4;
    (void)tiles_x;
}

// Hardware square root (MUFU, a few ulp) for the conservative filters below: they only need an
// upper bound on each chord's extent, so its error is absorbed by an extra outward margin of
// 1e-6 * h (>> the approximation error) on top of the fp32-rounding margins; unlike IEEE sqrtf it
// has no slow-path subroutine, so the filter stays in registers.
__device__ __forceinline__ float sqrt_approx(float x) {
    float r;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

// The same x-extent computation with the Span parameters precomputed in preprocess (rec2.w = sy,
// rec3 = (ky/(-qa), yc/(-qa), -qb/(2 qa), sx), sx < 0: box only): may the Gaussian produce a
// fragment at a pixel centre in [X0, X1] x [Y0, Y1]?  Conservative (the exact decision is the
// per-pixel spec); used by the raster's tile and warp filters.  The right (left) end of the
// ellipse's x-extent over the row band is at its rightmost (leftmost) point (+-sx, +-sy) when
// that lies in the band, else at the band edge nearest to it.
__device__ __forceinline__ bool band_relevant(float4 a, float4 e2, float4 e3, float X0, float X1, float Y0, float Y1) {
    const float mx = a.x, my = a.y;
    if (my + e2.y < Y0 || my - e2.y > Y1) return false;
    float xl = mx - e2.x, xr = mx + e2.x;
    const float sx = e3.w, sy = e2.w;
    if (sx > 0.f) {
        const float ey0 = Y0 - 0.5f - my, ey1 = Y1 + 0.5f - my;
        // right end: the band edge nearest to the rightmost point (or the point itself)
        const float eyr = fminf(fmaxf(sy, ey0), ey1), eyl = fminf(fmaxf(-sy, ey0), ey1);
        const float h2r = e3.x * eyr * eyr - e3.y, h2l = e3.x * eyl * eyl - e3.y;
        const bool inr = sy >= ey0 && sy <= ey1, inl = -sy >= ey0 && -sy <= ey1;
        if ((!inr && h2r < 0.f) || (!inl && h2l < 0.f)) return false;  // the band misses the ellipse
        const float hr = sqrt_approx(fmaxf(h2r, 0.f)), hl = sqrt_approx(fmaxf(h2l, 0.f));
        const float rr = inr ? sx : e3.z * eyr + hr;
        const float ll = inl ? -sx : e3.z * eyl - hl;
        xr = fminf(xr, mx + rr + 0.5f + 1e-4f * (fabsf(rr) + fabsf(mx)) + 1e-6f * hr + 1e-3f);
        xl = fmaxf(xl, mx + ll - 0.5f - 1e-4f * (fabsf(ll) + fabsf(mx)) - 1e-6f * hl - 1e-3f);
        if (!(xl <= xr)) return false;
    }
    return xr >= X0 && xl <= X1;
}

// DESIGN.md §3 exp2_spec for ycut <= y <= 0 (the caller's conservative prune guarantees
// y >= ycut > -64, so the oracle's y < -64 branch is unreachable here).
__device__ __forceinline__ float exp2_spec(float y) {
    const float magic = 0x1.8p23f;
    float t = __fadd_rn(y, magic);  // round-half-even to an integer
    float kf = __fsub_rn(t, magic);
    float f = __fsub_rn(y, kf);
    float p = 0x1.5bba14p-10f;
    p = __fmaf_rn(p, f, 0x1.3cea88p-7f);
    p = __fmaf_rn(p, f, 0x1.c6b752p-5f);
    p = __fmaf_rn(p, f, 0x1.ebf9bcp-3f);
    p = __fmaf_rn(p, f, 0x1.62e42ap-1f);
    p = __fmaf_rn(p, f, 1.0f);
    // ldexp(p, k): bits(t) << 23 == k << 23 (mod 2^32) for t = 1.5*2^23 + k
    return __int_as_float(__float_as_int(p) + (__float_as_int(t) << 23));
}

// One pixel of DESIGN.md §3 step PX for the record (a = mx, my, r, o; b = qa, qb, qc, ycut):
// returns e (0 when the fragment does not contribute) and updates T (0 = finished pixel).
// `live` gates the record (warp mask bit).  Shared by the uplift and render kernels.
__device__ __forceinline__ float pixel_fragment(const float4& a, const float4& b, float px, float py, bool live,
                                                float& T, bool& con) {
    const float dx = __fsub_rn(px, a.x), dy = __fsub_rn(py, a.y);
    const bool sq = live && fabsf(dx) <= a.z && fabsf(dy) <= a.z;
    const float q = __fmaf_rn(dx, __fmaf_rn(b.x, dx, __fmul_rn(b.y, dy)), __fmul_rn(__fmul_rn(b.z, dy), dy));
    const float al = fminf(K_ACLAMP, __fmul_rn(a.w, exp2_spec(q)));
    const float Tn = __fmul_rn(T, __fsub_rn(1.0f, al));
    const bool pass = sq && !(q > 0.f) && q >= b.w && al >= K_AMIN;
    con = pass && !(Tn < K_TMIN);
    const float e = con ? __fmul_rn(al, T) : 0.f;
    T = con ? Tn : (pass ? 0.f : T);
    return e;
}

// fused cross-rank reduction + Top-K (kernels.cu): the P ranks' partial W (this level's base,
// [Npad, L] each), device-accessible pointers (local or CUDA IPC mappings)
constexpr int MAX_PEERS = 16;
struct PeerRows {
    const float* W[MAX_PEERS];
    int n;
};
void launch_topk_peers(const PeerRows& peers, int64_t first_row, int64_t rows, int64_t valid_rows, int L, int K,
                       uint32_t* atoms, float* coefs, cudaStream_t s);

// thread-local message returned by scoup_last_error() (api.cu)
void set_last_error(const char* msg);

// ---- decode (decode.cu): F = W_hat C on tcgen05 (3xTF32)
bool decode_tc_supported(int L, int D);
size_t decode_tc_scratch_bytes(int L, int D);
cudaError_t launch_decode_tc(const float* W_hat, int64_t P, int L, int D, const float* C, float* scratch, float* F,
                             int num_sms, cudaStream_t s);

// ---- paired FP32 (sm_100 FADD2 / FMUL2 / FFMA2): two independent IEEE round-to-nearest
// operations per instruction; a pair lives in a 64-bit register (lo = first element)
typedef unsigned long long f2;
__device__ __forceinline__ f2 f2_pack(float lo, float hi) {
    f2 r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
    return r;
}
__device__ __forceinline__ void f2_split(f2 v, float& lo, float& hi) {
    asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
__device__ __forceinline__ f2 f2_add(f2 a, f2 b) {
    f2 r;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ f2 f2_sub(f2 a, f2 b) {
    f2 r;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ f2 f2_mul(f2 a, f2 b) {
    f2 r;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ f2 f2_fma(f2 a, f2 b, f2 c) {
    f2 r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
    return r;
}
__device__ __forceinline__ f2 f2_rsub(f2 a, float s) { return f2_sub(f2_pack(s, s), a); }  // s - a
__device__ __forceinline__ f2 f2_fmac(f2 a, f2 b, float c) { return f2_fma(a, b, f2_pack(c, c)); }

// exp2_spec (internal.cuh) on a pair: the same operations element-wise.
__device__ __forceinline__ f2 exp2_spec2(f2 y) {
    const float magic = 0x1.8p23f;  // 1.5 * 2^23
    const f2 mg = f2_pack(magic, magic);
    const f2 t = f2_add(y, mg);
    const f2 kf = f2_sub(t, mg);
    const f2 f = f2_sub(y, kf);
    f2 p = f2_fmac(f2_pack(0x1.5bba14p-10f, 0x1.5bba14p-10f), f, 0x1.3cea88p-7f);
    p = f2_fmac(p, f, 0x1.c6b752p-5f);
    p = f2_fmac(p, f, 0x1.ebf9bcp-3f);
    p = f2_fmac(p, f, 0x1.62e42ap-1f);
    p = f2_fmac(p, f, 1.0f);
    float p0, p1, t0, t1;
    f2_split(p, p0, p1);
    f2_split(t, t0, t1);
    return f2_pack(__int_as_float(__float_as_int(p0) + (__float_as_int(t0) << 23)),
                   __int_as_float(__float_as_int(p1) + (__float_as_int(t1) << 23)));
}


// ---- launchers (kernels.cu) ----
void launch_activate(const float* means, const float* scales, const float* rots, const float* opac,
                     int64_t G, PackedGaussians pg, ErrorLatch err, cudaStream_t s);
void launch_bounds(PackedGaussians pg, int64_t G, int* bbox, cudaStream_t s);
void launch_depth_hist(PackedGaussians pg, int64_t G, const CamBatch& cams, int key_bits, uint32_t* hist,
                       cudaStream_t s);
void launch_depth_pass_near(PackedGaussians pg, int64_t G, const CamBatch& cams, int key_bits, const uint32_t* thr,
                            uint32_t* code, unsigned long long* visible_ctr, ErrorLatch err, const Binning& bn,
                            uint32_t* trect, uint32_t* counts, uint32_t* sel, int* nsel, cudaStream_t s);
// stable compactions into vb.sel / vb.nsel; temp storage grown through *tmp / *tmp_bytes
void launch_preprocess(PackedGaussians pg, int64_t G, const CamBatch& cams, Binning bn, ViewBuffers vb,
                       int key_bits, int64_t nsel, cudaStream_t s);
size_t binsort_segments_max(int64_t entries, int nv);
uint32_t binsort_segment_len(int64_t entries);
void binsort_set_segment_override(int len);
void launch_binsort_gather(const uint32_t* sval_sorted, const uint32_t* tiles, int64_t nsel, uint32_t* offs,
                           BsInfo* info, cudaStream_t s);
void launch_binsort(const uint32_t* sel_offsets, int tiles_per_view, const uint32_t* offs,
                    const uint32_t* sval_sorted, const uint2* rect, int64_t nsel, int64_t entries, int nv,
                    int bins_x, int nb, BsInfo* info, uint32_t* cnt, uint16_t* ebin, uint32_t* eel, uint2* ranges,
                    uint32_t* eval, cudaStream_t s);
int select_tiles_per_view(int64_t G);
// custom stable compactions (kernels.cu): near / far chunk selections into vb.sel, count into
// vb.nsel; counts = scratch of select_counts_needed(G, nviews) tile counts
size_t select_counts_needed(int64_t G, int nviews);
void launch_select_far2(const ViewBuffers& vb, PackedGaussians pg, int64_t G, int nviews, int key_bits,
                        const Binning& bn, uint32_t* counts, cudaStream_t s);
void launch_ingest_dense(const float* in, int64_t n, float* out, ErrorLatch err, cudaStream_t s);
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
    const float4* rec3;
    float* Tstate;                // [nviews * H*W] transmittance carried between chunks
    uint8_t* tile_live;           // [nviews * tiles]
    int chunk;                    // 0: first chunk (T starts at 1), else continue from Tstate
    bool count_tests;             // instrumented variant: count contributions and support tests
    bool dense;                   // dense features (Eq. 3 baseline): S == L, atom = slot, no atoms table
    // render mode (Eq. 7, launch_render): per-pixel sum of the stored K-sparse codes
    const uint32_t* r_atoms;      // [G, rK]
    const float* r_coefs;
    int rK;
    float* r_out;                 // [views, H, W, L]: the batch's views start at r_view0
    int64_t r_view0;
    int nlev;                            // semantic levels fused in this pass (1..MAX_LEV)
    const uint32_t* region_ids[MAX_VB][MAX_LEV];  // [H*W] per view and level
    int64_t code_row0[MAX_VB][MAX_LEV];  // first row of (view, level) in the combined code table
    int32_t num_regions[MAX_VB][MAX_LEV];
    long long pixel_base[MAX_VB];        // flat index of the view's first pixel (error reports)
    long long* contrib_out[MAX_VB];      // optional per-view counters
    const uint32_t* code_atoms;   // sanitised combined table (all levels), rows of S slots
    const float* code_coefs;
    int S;
    int L;
    float* W;                     // [nlev][W_level_stride]
    int64_t W_level_stride;       // rows_padded * L
    float* Z;
    unsigned long long* contrib_ctr;  // handle stats
    unsigned long long* support_ctr;  // handle stats: support tests
    unsigned long long* lane_eval_ctr;  // handle stats: lane evaluations (32 per warp-record)
    unsigned long long* red_ctr;  // handle stats: global reductions issued (lane level, W and Z)
    ErrorLatch err;
};
void launch_raster(const RasterParams& p, cudaStream_t s);
// two pixels per thread (raster2.cu): the single-level sparse-code path (nlev == 1, !dense)
bool raster2_supported(const RasterParams& p);
void launch_raster2(const RasterParams& p, cudaStream_t s);
void raster2_set_slots_override(int slots);  // 0: adaptive (scoup_diag_set_raster2_slots)
void launch_render(const RasterParams& p, cudaStream_t s);

void launch_topk(const float* W, int64_t rows, int64_t valid_rows, int L, int K, uint32_t* atoms, float* coefs,
                 float* entropy, cudaStream_t s);

}  // namespace scoup
