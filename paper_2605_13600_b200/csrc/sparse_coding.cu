// sparse_coding.cu -- 2D sparse coding of region features into SCOUP's region codes
// (Eq. 4; recipe P:97; C ABI in
// include/scoup_sparse_coding.h; readings R-SC1..R-SC7 in DESIGN.md §14).
//
// One epoch = two kernels, replayed from a captured CUDA graph:
//   sc_epoch_kernel     one warp per region (grid-stride), whole region in registers (lane l
//                       holds logits l, l+32, .. and features d = l, l+32, ..): soft top-K by K
//                       rounds of warp arg-max (ties -> lower index), the reconstruction
//                       x = sum_k w_k C_{a_k}, cos(x, f), the loss, d loss / d x, d loss / d w_k,
//                       d loss / d z (restricted softmax), and the Adam step of the region's own
//                       logits (no other region touches them).  The codebook gradient w_k g is
//                       added into a per-CTA accumulator [L, D] in shared memory and written out
//                       as the CTA's partial (no global atomics, deterministic reduction order).
//   sc_codebook_kernel  sums the CTA partials per codebook entry (coalesced), Adam step of C,
//                       the epoch's loss (block 0) and the step counter (last block).
// k-means: per seeding step a distance-update kernel, an fp64 inclusive scan (CUB) and a pick
// kernel; Lloyd iterations assign rows to the nearest centre (codebook in shared memory) and
// accumulate the new centres.
#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <cmath>
#include <string>

#include "../../include/scoup_sparse_coding.h"
#include "internal.cuh"

namespace scoup {
namespace {

constexpr unsigned FULL = 0xffffffffu;
// threads of the epoch kernel: 32 warps (one region at a time each) hide the dependent loads
// best; the wide instantiations (KMAX or DPL of 32) need more registers and run 16 warps
template <int DPL, int KMAX>
constexpr int sc_threads() { return (KMAX >= 32 || DPL >= 32) ? 512 : 1024; }
constexpr int MAX_DPL = 32;      // D <= 1024
constexpr int MAX_LPL = 4;       // L <= 128
constexpr int SC_MAX_K = 32;

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
    return v;
}

struct ScDev {
    const float* F;  // [R, D]
    float *Z, *mZ, *vZ;   // [R, L]
    float *C, *mC, *vC;   // [L, D]
    float* partials;      // [nblk, L*D]
    float* loss_part;     // [nblk]
    float* loss_hist;     // [epochs] of the current train call
    long long* step;      // Adam steps taken
    unsigned* ticket;     // last-block detection of the codebook kernel
    int64_t R;
    int D, L, K;
    float lr, b1, b2, eps;
    ErrorLatch err;
};

// K largest logits of the warp's region (ties -> lower index), in order; every lane gets the
// same sel/zs.  z: lane's logits at l = lane + 32 i (-inf past L).
template <int LPL, int KMAX>
__device__ __forceinline__ void warp_topk(const float (&z)[LPL], int K, int lane, int (&sel)[KMAX], float (&zs)[KMAX]) {
    unsigned taken = 0u;  // bit i: my entry i already selected
#pragma unroll
    for (int k = 0; k < KMAX; k++) {
        if (k >= K) {
            sel[k] = 0;
            zs[k] = -INFINITY;
            continue;
        }
        // the round's largest untaken logit (5 float shuffles), then its lowest index: the first
        // entry slot i whose ballot of (untaken and equal) is non-empty, lowest lane in it
        float bv = -INFINITY;
#pragma unroll
        for (int i = 0; i < LPL; i++)
            if (!((taken >> i) & 1u)) bv = fmaxf(bv, z[i]);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) bv = fmaxf(bv, __shfl_xor_sync(FULL, bv, o));
        int bi = -1;
#pragma unroll
        for (int i = 0; i < LPL; i++) {
            const unsigned b = __ballot_sync(FULL, !((taken >> i) & 1u) && z[i] == bv);
            if (bi < 0 && b) bi = (__ffs(b) - 1) + 32 * i;
        }
        if (bi < 0) {  // (non-finite logits only: the first untaken entry, never out of range)
#pragma unroll
            for (int i = LPL - 1; i >= 0; i--) {
                const unsigned b = __ballot_sync(FULL, !((taken >> i) & 1u));
                if (b) bi = (__ffs(b) - 1) + 32 * i;
            }
        }
        sel[k] = bi;
        zs[k] = bv;
        if ((bi & 31) == lane) taken |= 1u << (bi >> 5);
    }
}

template <int DPL, int LPL, int KMAX, int NT = sc_threads<DPL, KMAX>()>
__global__ void __launch_bounds__(NT) sc_epoch_kernel(ScDev p) {
    extern __shared__ float sgC[];  // [L * D] this CTA's codebook gradient
    __shared__ float sloss[NT / 32];
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const int D = p.D, L = p.L, K = p.K, LD = L * D;
    for (int i = t; i < LD; i += NT) sgC[i] = 0.f;
    __syncthreads();
    const long long step = *p.step + 1;
    const float bc1 = (float)(1.0 - pow((double)p.b1, (double)step));
    const float bc2 = (float)(1.0 - pow((double)p.b2, (double)step));
    const float invR = 1.0f / (float)p.R;
    float lossacc = 0.f;
    const int64_t nw = (int64_t)gridDim.x * (NT / 32);
    for (int64_t r = (int64_t)blockIdx.x * (NT / 32) + warp; r < p.R; r += nw) {
        float z[LPL];
#pragma unroll
        for (int i = 0; i < LPL; i++) {
            const int l = lane + 32 * i;
            z[i] = l < L ? p.Z[r * L + l] : -INFINITY;
        }
        int sel[KMAX];
        float zs[KMAX], w[KMAX];
        warp_topk<LPL, KMAX>(z, K, lane, sel, zs);
        // restricted softmax (zs[0] is the largest kept logit); slots past K have weight 0
        float wsum = 0.f;
#pragma unroll
        for (int k = 0; k < KMAX; k++) {
            w[k] = k < K ? expf(zs[k] - zs[0]) : 0.f;
            wsum += w[k];
        }
#pragma unroll
        for (int k = 0; k < KMAX; k++) w[k] /= wsum;
        // the kept codebook rows: re-read (L1/L2) for the backward pass, or kept in registers
        // when the 512-thread instantiation leaves room (KMAX * DPL <= 64)
        constexpr bool CACHE = NT <= 512 && KMAX * DPL <= 64;
        float cv[CACHE ? KMAX : 1][CACHE ? DPL : 1];
        const float* Cr = p.C;
        float f[DPL], x[DPL];
        float xf = 0.f, xx = 0.f, ff = 0.f;
#pragma unroll
        for (int i = 0; i < DPL; i++) {
            const int d = lane + 32 * i;
            f[i] = d < D ? __ldg(p.F + r * D + d) : 0.f;
            float acc = 0.f;
            if (d < D) {
#pragma unroll
                for (int k = 0; k < KMAX; k++)
                    if (k < K) {
                        const float c = __ldg(Cr + (int64_t)sel[k] * D + d);
                        if (CACHE) cv[CACHE ? k : 0][CACHE ? i : 0] = c;
                        acc = fmaf(w[k], c, acc);
                    }
            }
            x[i] = acc;
            xf = fmaf(acc, f[i], xf);
            xx = fmaf(acc, acc, xx);
            ff = fmaf(f[i], f[i], ff);
        }
        xf = warp_sum(xf);
        xx = warp_sum(xx);
        ff = warp_sum(ff);
        const float nx = fmaxf(sqrtf(xx), 1e-12f), nf = sqrtf(ff);
        if (!(nf > 0.f) || !isfinite(nf)) {
            if (lane == 0) latch_error(p.err, ERR_CODE, (long long)r);
            continue;
        }
        const float cs = xf / (nx * nf);
        lossacc += 1.0f - cs;  // (lane-uniform; lane 0's copy is summed)
        const float a1 = 1.0f / (nx * nf), a2 = cs / (nx * nx);
        float gw[KMAX];
#pragma unroll
        for (int k = 0; k < KMAX; k++) gw[k] = 0.f;
#pragma unroll
        for (int i = 0; i < DPL; i++) {
            const int d = lane + 32 * i;
            if (d >= D) continue;
            const float g = -(f[i] * a1 - a2 * x[i]) * invR;  // d loss / d x_d
#pragma unroll
            for (int k = 0; k < KMAX; k++) {
                if (k >= K) continue;
                const int ci = sel[k] * D + d;
                gw[k] = fmaf(g, CACHE ? cv[CACHE ? k : 0][CACHE ? i : 0] : __ldg(Cr + ci), gw[k]);
                atomicAdd(&sgC[ci], w[k] * g);  // d loss / d C_{a_k} += w_k g
            }
        }
        float s = 0.f;
#pragma unroll
        for (int k = 0; k < KMAX; k++) {
            if (k >= K) continue;
            gw[k] = warp_sum(gw[k]);
            s = fmaf(w[k], gw[k], s);
        }
        // Adam on the region's logits: kept entries get w_k (gw_k - s), the rest 0
#pragma unroll
        for (int i = 0; i < LPL; i++) {
            const int l = lane + 32 * i;
            if (l >= L) continue;
            float g = 0.f;
#pragma unroll
            for (int k = 0; k < KMAX; k++)
                if (k < K && sel[k] == l) g = w[k] * (gw[k] - s);
            const int64_t zi = r * L + l;
            const float m = p.b1 * p.mZ[zi] + (1.0f - p.b1) * g;
            const float v = p.b2 * p.vZ[zi] + (1.0f - p.b2) * g * g;
            p.mZ[zi] = m;
            p.vZ[zi] = v;
            p.Z[zi] = z[i] - p.lr * (m / bc1) / (sqrtf(v / bc2) + p.eps);
        }
    }
    if (lane == 0) sloss[warp] = lossacc;
    __syncthreads();
    if (t == 0) {
        float sl = 0.f;
        for (int i = 0; i < NT / 32; i++) sl += sloss[i];
        p.loss_part[blockIdx.x] = sl;
    }
    float* out = p.partials + (int64_t)blockIdx.x * LD;
    for (int i = t; i < LD; i += NT) out[i] = sgC[i];
}

__global__ void sc_codebook_kernel(ScDev p, int nblk) {
    const int LD = p.L * p.D;
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const long long step = *p.step + 1;
    if (i < LD) {
        // the CTA partials in a fixed order: four interleaved running sums keep many loads in
        // flight (the epoch stays deterministic)
        float g0 = 0.f, g1 = 0.f, g2 = 0.f, g3 = 0.f;
        int c = 0;
#pragma unroll 2
        for (; c + 4 <= nblk; c += 4) {
            g0 += __ldg(p.partials + (int64_t)c * LD + i);
            g1 += __ldg(p.partials + (int64_t)(c + 1) * LD + i);
            g2 += __ldg(p.partials + (int64_t)(c + 2) * LD + i);
            g3 += __ldg(p.partials + (int64_t)(c + 3) * LD + i);
        }
        for (; c < nblk; c++) g0 += __ldg(p.partials + (int64_t)c * LD + i);
        const float g = (g0 + g1) + (g2 + g3);
        const float bc1 = (float)(1.0 - pow((double)p.b1, (double)step));
        const float bc2 = (float)(1.0 - pow((double)p.b2, (double)step));
        const float m = p.b1 * p.mC[i] + (1.0f - p.b1) * g;
        const float v = p.b2 * p.vC[i] + (1.0f - p.b2) * g * g;
        p.mC[i] = m;
        p.vC[i] = v;
        p.C[i] -= p.lr * (m / bc1) / (sqrtf(v / bc2) + p.eps);
    }
    if (blockIdx.x == 0 && threadIdx.x < 32) {
        float s = 0.f;
        for (int c = threadIdx.x; c < nblk; c += 32) s += p.loss_part[c];
        s = warp_sum(s);
        if (threadIdx.x == 0) {
            const float loss = s / (float)p.R;
            if (p.loss_hist) p.loss_hist[step - 1] = loss;
            if (!isfinite(loss)) latch_error(p.err, ERR_CODE, -1 - (long long)(step - 1));
        }
    }
    // the last block to finish advances the step counter (every block read it above)
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        if (atomicAdd(p.ticket, 1u) == gridDim.x - 1) {
            *p.step = step;
            *p.ticket = 0u;
            __threadfence();
        }
    }
}

// z_{r,l} = 10 cos(f_r, C_l) (R-SC5); cnorm: |C_l| (floored).
template <int DPL>
__global__ void sc_init_logits_kernel(const float* F, const float* C, const float* cnorm, int64_t R, int D, int L,
                                      float* Z, float* mZ, float* vZ) {
    const int lane = threadIdx.x & 31;
    const int64_t nw = (int64_t)gridDim.x * (blockDim.x / 32);
    for (int64_t r = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5); r < R; r += nw) {
        float f[DPL], ff = 0.f;
#pragma unroll
        for (int i = 0; i < DPL; i++) {
            const int d = lane + 32 * i;
            f[i] = d < D ? F[r * D + d] : 0.f;
            ff = fmaf(f[i], f[i], ff);
        }
        const float nf = sqrtf(warp_sum(ff));
        for (int l = 0; l < L; l++) {
            float dot = 0.f;
#pragma unroll
            for (int i = 0; i < DPL; i++) {
                const int d = lane + 32 * i;
                if (d < D) dot = fmaf(f[i], C[(int64_t)l * D + d], dot);
            }
            dot = warp_sum(dot);
            if (lane == 0) {
                Z[r * L + l] = 10.0f * dot / (nf * cnorm[l]);
                mZ[r * L + l] = 0.f;
                vZ[r * L + l] = 0.f;
            }
        }
    }
}

__global__ void sc_row_norms_kernel(const float* C, int L, int D, float* norms) {
    const int l = blockIdx.x, lane = threadIdx.x;
    float s = 0.f;
    for (int d = lane; d < D; d += 32) s = fmaf(C[(int64_t)l * D + d], C[(int64_t)l * D + d], s);
    s = warp_sum(s);
    if (lane == 0) norms[l] = fmaxf(sqrtf(s), 1e-12f);
}

// Feature check: finite, non-zero rows (latched EDATA with the row).
__global__ void sc_check_features_kernel(const float* F, int64_t R, int D, ErrorLatch err) {
    const int lane = threadIdx.x & 31;
    const int64_t nw = (int64_t)gridDim.x * (blockDim.x / 32);
    for (int64_t r = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5); r < R; r += nw) {
        float s = 0.f;
        bool ok = true;
        for (int d = lane; d < D; d += 32) {
            const float v = F[r * D + d];
            ok = ok && isfinite(v);
            s += v * v;
        }
        s = warp_sum(s);
        ok = __all_sync(FULL, ok);
        if (lane == 0 && (!ok || !(s > 0.f))) latch_error(err, ERR_CODE, (long long)r);
    }
}

// ---- k-means (R-SC6)
// d2[r] = |f_r - c|^2 (first) or min(d2[r], |f_r - c|^2); also the fp64 copy for the scan.
__global__ void km_d2_kernel(const float* F, int64_t R, int D, const float* c, int first, float* d2, double* d2d) {
    const int lane = threadIdx.x & 31;
    const int64_t nw = (int64_t)gridDim.x * (blockDim.x / 32);
    for (int64_t r = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5); r < R; r += nw) {
        float s = 0.f;
        for (int d = lane; d < D; d += 32) {
            const float e = F[r * D + d] - c[d];
            s = fmaf(e, e, s);
        }
        s = warp_sum(s);
        if (lane == 0) {
            const float v = first ? s : fminf(d2[r], s);
            d2[r] = v;
            d2d[r] = (double)v;
        }
    }
}

// first row r with cum[r] > u * total (cum inclusive, nondecreasing); R-1 if none.
__global__ void km_pick_kernel(const double* cum, int64_t R, double u, int* pick) {
    const double total = cum[R - 1];
    const double thr = u * total;
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= R) return;
    const double prev = r == 0 ? 0.0 : cum[r - 1];
    if ((prev <= thr && cum[r] > thr) || (r == R - 1 && !(cum[r] > thr))) atomicMin(pick, (int)r);
}

__global__ void km_copy_kernel(const float* F, const double* cum, int64_t R, int D, const int* pick,
                               const float* fallback_row, float* dst) {
    const bool any = cum[R - 1] > 0.0;
    const int r = *pick;
    for (int d = threadIdx.x; d < D; d += blockDim.x) dst[d] = any ? F[(int64_t)r * D + d] : fallback_row[d];
}

// Lloyd assignment (ties -> lower index) + accumulation of the new centres.
template <int DPL>
__global__ void km_assign_kernel(const float* F, int64_t R, int D, int L, const float* C, int* assign, int* changed,
                                 float* sums, int* counts) {
    extern __shared__ float sC[];  // [L * D]
    for (int i = threadIdx.x; i < L * D; i += blockDim.x) sC[i] = C[i];
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int64_t nw = (int64_t)gridDim.x * (blockDim.x / 32);
    for (int64_t r = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5); r < R; r += nw) {
        float f[DPL];
#pragma unroll
        for (int i = 0; i < DPL; i++) {
            const int d = lane + 32 * i;
            f[i] = d < D ? F[r * D + d] : 0.f;
        }
        float best = INFINITY;
        int bi = 0;
        for (int l = 0; l < L; l++) {
            float s = 0.f;
#pragma unroll
            for (int i = 0; i < DPL; i++) {
                const int d = lane + 32 * i;
                if (d < D) {
                    const float e = f[i] - sC[l * D + d];
                    s = fmaf(e, e, s);
                }
            }
            s = warp_sum(s);
            if (s < best) {
                best = s;
                bi = l;
            }
        }
        if (lane == 0) {
            if (assign[r] != bi) *changed = 1;
            assign[r] = bi;
            atomicAdd(&counts[bi], 1);
        }
#pragma unroll
        for (int i = 0; i < DPL; i++) {
            const int d = lane + 32 * i;
            if (d < D) atomicAdd(&sums[(int64_t)bi * D + d], f[i]);
        }
    }
}

__global__ void km_update_kernel(float* C, const float* sums, const int* counts, int L, int D) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= L * D) return;
    const int c = counts[i / D];
    if (c > 0) C[i] = sums[i] / (float)c;
}

// Hard codes (R-SC7).
template <int LPL>
__global__ void sc_encode_kernel(const float* Z, int64_t R, int L, int K, uint32_t* atoms, float* coefs) {
    const int lane = threadIdx.x & 31;
    const int64_t nw = (int64_t)gridDim.x * (blockDim.x / 32);
    for (int64_t r = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5); r < R; r += nw) {
        float z[LPL];
#pragma unroll
        for (int i = 0; i < LPL; i++) {
            const int l = lane + 32 * i;
            z[i] = l < L ? Z[r * L + l] : -INFINITY;
        }
        int sel[SC_MAX_K];
        float zs[SC_MAX_K];
        warp_topk<LPL, SC_MAX_K>(z, K, lane, sel, zs);
        float ws = 0.f;
#pragma unroll
        for (int k = 0; k < SC_MAX_K; k++) ws += k < K ? expf(zs[k] - zs[0]) : 0.f;
        if (lane < K) {
            float zk = 0.f;
            int ak = 0;
#pragma unroll
            for (int k = 0; k < SC_MAX_K; k++)
                if (k == lane) {
                    zk = zs[k];
                    ak = sel[k];
                }
            atoms[r * K + lane] = (uint32_t)ak;
            coefs[r * K + lane] = expf(zk - zs[0]) / ws;
        }
    }
}

template <typename F>
void dispatch_dpl(int D, F&& f) {
    const int dpl = (D + 31) / 32;
    if (dpl <= 4) f(std::integral_constant<int, 4>{});
    else if (dpl <= 16) f(std::integral_constant<int, 16>{});
    else f(std::integral_constant<int, 32>{});
}

template <typename F>
void dispatch_lpl(int L, F&& f) {
    if (L <= 64) f(std::integral_constant<int, 2>{});
    else f(std::integral_constant<int, 4>{});
}

}  // namespace
}  // namespace scoup

using namespace scoup;

struct scoup_sc {
    int device = 0;
    cudaStream_t stream = nullptr;
    int64_t R = 0;
    int D = 0, L = 0, K = 0;
    const float* F = nullptr;
    float *C = nullptr, *Z = nullptr, *mC = nullptr, *vC = nullptr, *mZ = nullptr, *vZ = nullptr;
    float *partials = nullptr, *loss_part = nullptr;
    long long* step = nullptr;
    unsigned* ticket = nullptr;
    int* err_code = nullptr;
    long long* err_index = nullptr;
    int nblk = 0;
    size_t epoch_smem = 0;
    bool latched = false;
};

namespace {

#define SCK(expr)                                                                                  \
    do {                                                                                           \
        cudaError_t _e = (expr);                                                                   \
        if (_e != cudaSuccess) {                                                                   \
            set_last_error((std::string("CUDA error in ") + #expr + ": " + cudaGetErrorString(_e)).c_str()); \
            return _e == cudaErrorMemoryAllocation ? SCOUP_ENOMEM : SCOUP_ECUDA;                   \
        }                                                                                          \
    } while (0)

scoup_status sc_fail(scoup_status st, const std::string& m) {
    set_last_error(m.c_str());
    return st;
}

struct DevGuard {
    int prev = -1;
    explicit DevGuard(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev) cudaSetDevice(dev);
    }
    ~DevGuard() {
        if (prev >= 0) cudaSetDevice(prev);
    }
};

bool dev_ptr(const void* p) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

ErrorLatch latch(scoup_sc* h) { return ErrorLatch{h->err_code, h->err_index}; }

scoup_status sc_check(scoup_sc* h) {
    int code = 0;
    long long idx = 0;
    SCK(cudaStreamSynchronize(h->stream));
    SCK(cudaMemcpy(&code, h->err_code, sizeof(int), cudaMemcpyDeviceToHost));
    if (!code) return SCOUP_OK;
    SCK(cudaMemcpy(&idx, h->err_index, sizeof(long long), cudaMemcpyDeviceToHost));
    h->latched = true;
    if (idx < 0) return sc_fail(SCOUP_EDATA, "sparse coding: non-finite loss at epoch " + std::to_string(-1 - idx));
    return sc_fail(SCOUP_EDATA, "sparse coding: region " + std::to_string(idx) +
                                    " has a zero or non-finite feature row");
}

ScDev make_dev(scoup_sc* h, float lr, float b1, float b2, float eps, float* loss_hist) {
    ScDev p{};
    p.F = h->F;
    p.Z = h->Z;
    p.mZ = h->mZ;
    p.vZ = h->vZ;
    p.C = h->C;
    p.mC = h->mC;
    p.vC = h->vC;
    p.partials = h->partials;
    p.loss_part = h->loss_part;
    p.loss_hist = loss_hist;
    p.step = h->step;
    p.ticket = h->ticket;
    p.R = h->R;
    p.D = h->D;
    p.L = h->L;
    p.K = h->K;
    p.lr = lr;
    p.b1 = b1;
    p.b2 = b2;
    p.eps = eps;
    p.err = latch(h);
    return p;
}

template <typename F>
void dispatch_kmax(int K, F&& f) {
    if (K <= 4) f(std::integral_constant<int, 4>{});
    else if (K <= 8) f(std::integral_constant<int, 8>{});
    else f(std::integral_constant<int, 32>{});
}

// launch (prepare = true: only set the kernel's shared-memory attribute, outside any capture)
void launch_epoch(scoup_sc* h, const ScDev& p, bool prepare = false) {
    dispatch_dpl(h->D, [&](auto dpl) {
        dispatch_lpl(h->L, [&](auto lpl) {
            dispatch_kmax(h->K, [&](auto km) {
                constexpr int DPL_ = decltype(dpl)::value, KM_ = decltype(km)::value;
                auto kern = sc_epoch_kernel<DPL_, decltype(lpl)::value, KM_>;
                if (prepare)
                    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)h->epoch_smem);
                else
                    kern<<<h->nblk, sc_threads<DPL_, KM_>(), h->epoch_smem, h->stream>>>(p);
            });
        });
    });
    if (prepare) return;
    const int LD = h->L * h->D;
    sc_codebook_kernel<<<(LD + 255) / 256, 256, 0, h->stream>>>(p, h->nblk);
}

scoup_status init_logits(scoup_sc* h) {
    float* norms = nullptr;
    SCK(cudaMallocAsync((void**)&norms, sizeof(float) * h->L, h->stream));
    sc_row_norms_kernel<<<h->L, 32, 0, h->stream>>>(h->C, h->L, h->D, norms);
    const int blocks = (int)std::min<int64_t>((h->R + 7) / 8, 4096);
    dispatch_dpl(h->D, [&](auto dpl) {
        sc_init_logits_kernel<decltype(dpl)::value>
            <<<blocks, 256, 0, h->stream>>>(h->F, h->C, norms, h->R, h->D, h->L, h->Z, h->mZ, h->vZ);
    });
    SCK(cudaMemsetAsync(h->mC, 0, sizeof(float) * h->L * h->D, h->stream));
    SCK(cudaMemsetAsync(h->vC, 0, sizeof(float) * h->L * h->D, h->stream));
    SCK(cudaMemsetAsync(h->step, 0, sizeof(long long), h->stream));
    SCK(cudaFreeAsync(norms, h->stream));
    SCK(cudaGetLastError());
    return SCOUP_OK;
}

}  // namespace

extern "C" {

scoup_status scoup_sc_init(int device, void* cuda_stream, int64_t R, int32_t D, int32_t L, int32_t K,
                           const float* features, scoup_sc** out) {
    set_last_error("");
    if (!out || !features) return sc_fail(SCOUP_EINVAL, "NULL argument");
    *out = nullptr;
    if (R < 1 || D < 1 || L < 1 || K < 1 || K > L) return sc_fail(SCOUP_EINVAL, "need R, D, L >= 1 and 1 <= K <= L");
    if (L > 32 * MAX_LPL || D > 32 * MAX_DPL || K > SC_MAX_K || (int64_t)L * D > 49152)
        return sc_fail(SCOUP_EUNSUPPORTED, "sparse coding limits: L <= 128, D <= 1024, K <= 32, L*D <= 49152");
    if (R > (int64_t)1 << 40) return sc_fail(SCOUP_EUNSUPPORTED, "R too large");
    DevGuard g(device);
    if (!dev_ptr(features)) return sc_fail(SCOUP_EINVAL, "features must be device memory");
    scoup_sc* h = new scoup_sc();
    h->device = device;
    h->stream = (cudaStream_t)cuda_stream;
    h->R = R;
    h->D = D;
    h->L = L;
    h->K = K;
    h->F = features;
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    const int64_t LD = (int64_t)L * D;
    h->epoch_smem = sizeof(float) * (size_t)LD;
    // one CTA per SM (the shared-memory accumulator); no more CTAs than 16-region groups
    h->nblk = (int)std::max<int64_t>(1, std::min<int64_t>(sms, (R + 15) / 16));
    auto al = [&](void** p, size_t bytes) { return cudaMallocAsync(p, std::max<size_t>(bytes, 4), h->stream); };
    cudaError_t e = cudaSuccess;
    for (float** q : {&h->C, &h->mC, &h->vC})
        if (e == cudaSuccess) e = al((void**)q, sizeof(float) * LD);
    for (float** q : {&h->Z, &h->mZ, &h->vZ})
        if (e == cudaSuccess) e = al((void**)q, sizeof(float) * R * L);
    if (e == cudaSuccess) e = al((void**)&h->partials, sizeof(float) * LD * h->nblk);
    if (e == cudaSuccess) e = al((void**)&h->loss_part, sizeof(float) * h->nblk);
    if (e == cudaSuccess) e = al((void**)&h->step, sizeof(long long));
    if (e == cudaSuccess) e = al((void**)&h->ticket, sizeof(unsigned));
    if (e == cudaSuccess) e = al((void**)&h->err_code, sizeof(int));
    if (e == cudaSuccess) e = al((void**)&h->err_index, sizeof(long long));
    if (e != cudaSuccess) {
        scoup_sc_free(h);
        return sc_fail(e == cudaErrorMemoryAllocation ? SCOUP_ENOMEM : SCOUP_ECUDA, cudaGetErrorString(e));
    }
    cudaMemsetAsync(h->ticket, 0, sizeof(unsigned), h->stream);
    cudaMemsetAsync(h->step, 0, sizeof(long long), h->stream);
    cudaMemsetAsync(h->err_code, 0, sizeof(int), h->stream);
    for (float* q : {h->C, h->mC, h->vC}) cudaMemsetAsync(q, 0, sizeof(float) * LD, h->stream);
    for (float* q : {h->Z, h->mZ, h->vZ}) cudaMemsetAsync(q, 0, sizeof(float) * R * L, h->stream);
    sc_check_features_kernel<<<(int)std::min<int64_t>((R + 7) / 8, 4096), 256, 0, h->stream>>>(features, R, D,
                                                                                                latch(h));
    e = cudaGetLastError();
    if (e != cudaSuccess) {
        scoup_sc_free(h);
        return sc_fail(SCOUP_ECUDA, cudaGetErrorString(e));
    }
    *out = h;
    return SCOUP_OK;
}

scoup_status scoup_sc_kmeans(scoup_sc* h, const double* uniforms, const float* fallback, int32_t max_iter,
                             int32_t* iters_out) {
    set_last_error("");
    if (!h || !uniforms || !fallback) return sc_fail(SCOUP_EINVAL, "NULL argument");
    if (max_iter < 0) return sc_fail(SCOUP_EINVAL, "max_iter < 0");
    if (h->latched) return sc_fail(SCOUP_ESTATE, "a latched data error is pending");
    DevGuard g(h->device);
    const int64_t R = h->R;
    const int D = h->D, L = h->L;
    for (int j = 0; j < L; j++)
        if (!(uniforms[j] >= 0.0 && uniforms[j] < 1.0)) return sc_fail(SCOUP_EINVAL, "uniforms must lie in [0, 1)");
    scoup_status st = sc_check(h);  // feature check first
    if (st != SCOUP_OK) return st;
    float *d2 = nullptr, *fb = nullptr, *sums = nullptr;
    double *d2d = nullptr, *cum = nullptr;
    int *pick = nullptr, *assign = nullptr, *changed = nullptr, *counts = nullptr;
    void* tmp = nullptr;
    size_t tmp_bytes = 0;
    cub::DeviceScan::InclusiveSum(nullptr, tmp_bytes, (double*)nullptr, (double*)nullptr, (int)R);
    SCK(cudaMallocAsync((void**)&d2, sizeof(float) * R, h->stream));
    SCK(cudaMallocAsync((void**)&d2d, sizeof(double) * R, h->stream));
    SCK(cudaMallocAsync((void**)&cum, sizeof(double) * R, h->stream));
    SCK(cudaMallocAsync((void**)&fb, sizeof(float) * L * D, h->stream));
    SCK(cudaMallocAsync((void**)&pick, sizeof(int), h->stream));
    SCK(cudaMallocAsync(&tmp, std::max<size_t>(tmp_bytes, 16), h->stream));
    SCK(cudaMemcpyAsync(fb, fallback, sizeof(float) * L * D, cudaMemcpyDefault, h->stream));
    // ---- k-means++ seeding
    const int wblocks = (int)std::min<int64_t>((R + 7) / 8, 4096);
    const int64_t r0 = std::min<int64_t>((int64_t)std::floor(uniforms[0] * (double)R), R - 1);
    SCK(cudaMemcpyAsync(h->C, h->F + r0 * D, sizeof(float) * D, cudaMemcpyDeviceToDevice, h->stream));
    for (int j = 0; j < L; j++) {
        km_d2_kernel<<<wblocks, 256, 0, h->stream>>>(h->F, R, D, h->C + (int64_t)j * D, j == 0, d2, d2d);
        if (j + 1 == L) break;
        SCK(cub::DeviceScan::InclusiveSum(tmp, tmp_bytes, d2d, cum, (int)R, h->stream));
        const int big = 0x7fffffff;
        SCK(cudaMemcpyAsync(pick, &big, sizeof(int), cudaMemcpyHostToDevice, h->stream));
        km_pick_kernel<<<(int)((R + 255) / 256), 256, 0, h->stream>>>(cum, R, uniforms[j + 1], pick);
        km_copy_kernel<<<1, 256, 0, h->stream>>>(h->F, cum, R, D, pick, fb + (int64_t)(j + 1) * D,
                                                 h->C + (int64_t)(j + 1) * D);
    }
    // ---- Lloyd
    SCK(cudaMallocAsync((void**)&assign, sizeof(int) * R, h->stream));
    SCK(cudaMallocAsync((void**)&changed, sizeof(int), h->stream));
    SCK(cudaMallocAsync((void**)&counts, sizeof(int) * L, h->stream));
    SCK(cudaMallocAsync((void**)&sums, sizeof(float) * L * D, h->stream));
    SCK(cudaMemsetAsync(assign, 0xff, sizeof(int) * R, h->stream));  // -1: no assignment yet
    const size_t asmem = sizeof(float) * (size_t)L * D;
    int it = 0;
    for (int iter = 0; iter <= max_iter; iter++) {
        SCK(cudaMemsetAsync(changed, 0, sizeof(int), h->stream));
        SCK(cudaMemsetAsync(counts, 0, sizeof(int) * L, h->stream));
        SCK(cudaMemsetAsync(sums, 0, sizeof(float) * L * D, h->stream));
        dispatch_dpl(D, [&](auto dpl) {
            auto kern = km_assign_kernel<decltype(dpl)::value>;
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)asmem);
            kern<<<wblocks, 256, asmem, h->stream>>>(h->F, R, D, L, h->C, assign, changed, sums, counts);
        });
        int ch = 0;
        SCK(cudaMemcpyAsync(&ch, changed, sizeof(int), cudaMemcpyDeviceToHost, h->stream));
        SCK(cudaStreamSynchronize(h->stream));
        if (!ch || iter == max_iter) break;  // the assignment is a fixpoint (or out of budget)
        km_update_kernel<<<(L * D + 255) / 256, 256, 0, h->stream>>>(h->C, sums, counts, L, D);
        it++;
    }
    if (iters_out) *iters_out = it;
    for (void* q : {(void*)d2, (void*)d2d, (void*)cum, (void*)fb, (void*)pick, tmp, (void*)assign, (void*)changed,
                    (void*)counts, (void*)sums})
        cudaFreeAsync(q, h->stream);
    SCK(cudaGetLastError());
    st = init_logits(h);
    if (st != SCOUP_OK) return st;
    return sc_check(h);
}

scoup_status scoup_sc_set_state(scoup_sc* h, const float* C, const float* Z, const float* mC, const float* vC,
                                const float* mZ, const float* vZ, int64_t t) {
    set_last_error("");
    if (!h) return sc_fail(SCOUP_EINVAL, "NULL handle");
    if (t < 0) return sc_fail(SCOUP_EINVAL, "t < 0");
    DevGuard g(h->device);
    const size_t LD = sizeof(float) * (size_t)h->L * h->D, RL = sizeof(float) * (size_t)h->R * h->L;
    const float* src[6] = {C, Z, mC, vC, mZ, vZ};
    float* dst[6] = {h->C, h->Z, h->mC, h->vC, h->mZ, h->vZ};
    const size_t bytes[6] = {LD, RL, LD, LD, RL, RL};
    for (int i = 0; i < 6; i++)
        if (src[i]) SCK(cudaMemcpyAsync(dst[i], src[i], bytes[i], cudaMemcpyDefault, h->stream));
    const long long tt = (long long)t;
    SCK(cudaMemcpyAsync(h->step, &tt, sizeof(long long), cudaMemcpyHostToDevice, h->stream));
    SCK(cudaStreamSynchronize(h->stream));
    return SCOUP_OK;
}

scoup_status scoup_sc_get_state(scoup_sc* h, float** C, float** Z, float** mC, float** vC, float** mZ, float** vZ,
                                int64_t* t) {
    set_last_error("");
    if (!h) return sc_fail(SCOUP_EINVAL, "NULL handle");
    DevGuard g(h->device);
    if (C) *C = h->C;
    if (Z) *Z = h->Z;
    if (mC) *mC = h->mC;
    if (vC) *vC = h->vC;
    if (mZ) *mZ = h->mZ;
    if (vZ) *vZ = h->vZ;
    if (t) {
        long long tt = 0;
        SCK(cudaMemcpyAsync(&tt, h->step, sizeof(long long), cudaMemcpyDeviceToHost, h->stream));
        SCK(cudaStreamSynchronize(h->stream));
        *t = tt;
    }
    return SCOUP_OK;
}

scoup_status scoup_sc_train(scoup_sc* h, int32_t epochs, float lr, float beta1, float beta2, float eps,
                            float* loss_out) {
    set_last_error("");
    if (!h) return sc_fail(SCOUP_EINVAL, "NULL handle");
    if (epochs < 0 || !(lr > 0.f) || !(beta1 >= 0.f && beta1 < 1.f) || !(beta2 >= 0.f && beta2 < 1.f) || !(eps >= 0.f))
        return sc_fail(SCOUP_EINVAL, "bad training hyper-parameters");
    if (h->latched) return sc_fail(SCOUP_ESTATE, "a latched data error is pending");
    if (epochs == 0) return SCOUP_OK;
    DevGuard g(h->device);
    // the loss history is indexed by the global step: a device buffer covering [0, t + epochs)
    long long t0 = 0;
    SCK(cudaMemcpyAsync(&t0, h->step, sizeof(long long), cudaMemcpyDeviceToHost, h->stream));
    SCK(cudaStreamSynchronize(h->stream));
    float* hist = nullptr;
    SCK(cudaMallocAsync((void**)&hist, sizeof(float) * (size_t)(t0 + epochs), h->stream));
    const ScDev p = make_dev(h, lr, beta1, beta2, eps, hist);
    launch_epoch(h, p, true);
    // capture a chunk of epochs once, replay it; the remainder launches directly
    const int chunk = std::min(epochs, 50);
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    cudaStream_t cs = nullptr;
    SCK(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
    cudaEvent_t ev = nullptr;
    SCK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    SCK(cudaEventRecord(ev, h->stream));
    SCK(cudaStreamWaitEvent(cs, ev, 0));
    cudaStream_t saved = h->stream;
    h->stream = cs;
    SCK(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
    for (int e = 0; e < chunk; e++) launch_epoch(h, p);
    cudaError_t ce = cudaStreamEndCapture(cs, &graph);
    h->stream = saved;
    if (ce != cudaSuccess) {
        cudaStreamDestroy(cs);
        cudaEventDestroy(ev);
        return sc_fail(SCOUP_ECUDA, std::string("graph capture: ") + cudaGetErrorString(ce));
    }
    SCK(cudaGraphInstantiate(&exec, graph, 0));
    for (int done = 0; done + chunk <= epochs; done += chunk) SCK(cudaGraphLaunch(exec, cs));
    h->stream = cs;
    for (int e = 0; e < epochs % chunk; e++) launch_epoch(h, p);
    h->stream = saved;
    SCK(cudaEventRecord(ev, cs));
    SCK(cudaStreamWaitEvent(h->stream, ev, 0));
    if (loss_out)
        SCK(cudaMemcpyAsync(loss_out, hist + t0, sizeof(float) * epochs, cudaMemcpyDefault, h->stream));
    SCK(cudaFreeAsync(hist, h->stream));
    SCK(cudaGetLastError());
    SCK(cudaStreamSynchronize(h->stream));
    cudaGraphExecDestroy(exec);
    cudaGraphDestroy(graph);
    cudaStreamDestroy(cs);
    cudaEventDestroy(ev);
    return sc_check(h);
}

scoup_status scoup_sc_encode(scoup_sc* h, uint32_t* atoms, float* coefs) {
    set_last_error("");
    if (!h || !atoms || !coefs) return sc_fail(SCOUP_EINVAL, "NULL argument");
    DevGuard g(h->device);
    if (!dev_ptr(atoms) || !dev_ptr(coefs)) return sc_fail(SCOUP_EINVAL, "atoms / coefs must be device memory");
    const int blocks = (int)std::min<int64_t>((h->R + 7) / 8, 4096);
    dispatch_lpl(h->L, [&](auto lpl) {
        sc_encode_kernel<decltype(lpl)::value><<<blocks, 256, 0, h->stream>>>(h->Z, h->R, h->L, h->K, atoms, coefs);
    });
    SCK(cudaGetLastError());
    return SCOUP_OK;
}

void scoup_sc_free(scoup_sc* h) {
    if (!h) return;
    DevGuard g(h->device);
    cudaStreamSynchronize(h->stream);
    for (void* q : {(void*)h->C, (void*)h->Z, (void*)h->mC, (void*)h->vC, (void*)h->mZ, (void*)h->vZ,
                    (void*)h->partials, (void*)h->loss_part, (void*)h->step, (void*)h->ticket, (void*)h->err_code,
                    (void*)h->err_index})
        if (q) cudaFree(q);
    delete h;
}

}  // extern "C"
