// decode.cu -- codebook decode F = W_hat C (Eq. 8)
// on the 5th-generation tensor cores.
//
// F [P, D] = W_hat [P, L] . C [L, D], fp32 in and out.  The contraction is short (K = L <= 64)
// and the output is wide (D = 512 floats per pixel), so the op is bound by writing F to HBM;
// plain fp32 FFMA cannot keep up with that write stream, tcgen05 can.  To keep fp32 accuracy on
// the tf32 tensor path every operand x is split exactly into x = big + small, big = x with the
// low 13 mantissa bits cleared (a tf32 value), small = x - big (exact in fp32, <= 13 significant
// bits), and the tile is accumulated as
//     D = A_big B_big + A_big B_small + A_small B_big          ("3xTF32")
// in fp32 in tensor memory: the dropped A_small B_small term and the tf32 reading of `small` are
// both below 2^-20 relative per product, i.e. the result matches an fp32 GEMM to ~1e-6.
//
// One persistent CTA per SM (12 warps, warp-specialised), a fixed N tile of NT = 256 columns of F
// (B = C^T[NT, L] split big/small, resident in shared memory), looping over 128-row M tiles:
//   * 8 producer warps: each A tile (128 x L fp32) is split and written to shared memory in the
//     K-major no-swizzle canonical UMMA layout (core matrices of 8 rows x 16 B; LBO = 128 B,
//     SBO = chunks-per-row * 128 B, which makes the layout linear in the 16-byte chunk index, so
//     the stores are contiguous).  The tile is handled in K parts with their own smem regions
//     and "part free" mbarriers, so the split of part p of tile i+1 overlaps the MMAs of the other
//     parts of tile i; each part's global loads are issued one tile ahead.  One thread issues the
//     3 (L / 8) tcgen05.mma (M=128, N=NT, K=8, kind::tf32) of a part into one of two 256-column
//     accumulator stages in TMEM and commits them to the mbarriers.
//   * 4 epilogue warps (one per TMEM lane quarter): tcgen05.ld 32x32b of a drained stage ->
//     registers -> a 32 x 32 fp32 block in shared memory in the TMA 128-byte-swizzle layout ->
//     one cp.async.bulk.tensor store per block (the TMA engine writes F; rows past P are clipped
//     by the tensor map), then an arrive on the stage's "empty" mbarrier.
// Measured (outdoor, 1600 x 1066 px, L = 64, D = 512): ~0.75 ms per view, 5.2 TB/s of HBM
// traffic (the F write stream dominates), vs 2.7 ms for cuBLAS SGEMM.
#include <cuda.h>
#include <cudaTypedefs.h>

#include "internal.cuh"

namespace scoup {

namespace {

constexpr int DM = 128;           // rows per M tile (UMMA M)
#ifndef DEC_NPROD
#define DEC_NPROD 8
#endif
constexpr int NUM_PROD = DEC_NPROD;            // producer warps (A split + MMA issue)
constexpr int NUM_EPI = 4;                     // epilogue warps (1 per TMEM lane quarter)
#ifndef DEC_NB
#define DEC_NB 2
#endif
constexpr int NB = DEC_NB;                     // TMA-store staging blocks per epilogue warp
constexpr int DEC_THREADS = 32 * (NUM_PROD + NUM_EPI);

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// tcgen05 shared-memory matrix descriptor: K-major, no swizzle, version 1 (sm_100).
__device__ __forceinline__ uint64_t umma_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    return (uint64_t)((addr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46);
}

__device__ __forceinline__ float tf32_big(float x) { return __uint_as_float(__float_as_uint(x) & 0xFFFFE000u); }

__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    uint32_t ok = 0;
    while (!ok) {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(ok)
            : "r"(bar), "r"(parity)
            : "memory");
    }
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}"
        :
        : "r"(tmem_d), "l"(da), "l"(db), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// 32 consecutive accumulator columns of this thread's TMEM lane (asynchronous: tmem_wait_ld)
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "
        "%14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
          "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
          "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// C [L, D] row-major -> C^T split into big / small, each [D/NT tiles][NT rows][L] in the K-major
// no-swizzle canonical layout (byte offset of (r, k) in a tile: (r/8)(L/4)128 + (k/4)128 +
// (r%8)16 + (k%4)4), so a tile is one contiguous block the decode kernel copies as is.
__global__ void decode_prep_kernel(const float* __restrict__ C, int L, int D, int NT, float* Bbig, float* Bsmall) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= L * D) return;
    const int k = i / D, n = i - k * D;
    const float x = C[i];
    const float big = tf32_big(x);
    const int nt = n / NT, r = n - nt * NT;
    const int64_t off = (int64_t)nt * NT * L + ((r >> 3) * (L / 4) * 32 + (k >> 2) * 32 + (r & 7) * 4 + (k & 3));
    Bbig[off] = big;
    Bsmall[off] = __fsub_rn(x, big);
}

template <int L>
__global__ void __launch_bounds__(DEC_THREADS, 1)
    decode_kernel(const float* __restrict__ A, int64_t P, int D, int NT, const float* __restrict__ Bbig,
                  const float* __restrict__ Bsmall, const __grid_constant__ CUtensorMap tmap_F) {
    extern __shared__ __align__(1024) unsigned char dsm[];
    const int nN = D / NT;
    const int n_tile = blockIdx.x % nN;
    const int64_t mtiles = (P + DM - 1) / DM;
    const int64_t mstep = gridDim.x / nN;
    const int64_t m0 = blockIdx.x / nN;
    float* sBb = reinterpret_cast<float*>(dsm);
    float* sBs = sBb + NT * L;
    float* sAb = sBs + NT * L;
    float* sAs = sAb + DM * L;
    // staging (TMA-store sources, 1024-byte aligned for the 128-byte swizzle): 2 x 4 KB per
    // epilogue warp; then the barriers: [0..3] A part free (its MMAs done), [4..5] accumulator
    // stage full, [6..7] stage drained by the epilogue warps (count NUM_EPI)
    float* stg_base = sAs + DM * L;
    uint64_t* bars = reinterpret_cast<uint64_t*>(stg_base + NUM_EPI * NB * 1024);
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 8);
    const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
    const uint32_t b_afree0 = smem_u32(bars), b_full0 = smem_u32(bars + 4), b_empty0 = smem_u32(bars + 6);

    // ---- B tile (this CTA's NT columns of F) -> shared memory, barriers, TMEM (512 columns)
    {
        const int4* gb = reinterpret_cast<const int4*>(Bbig + (int64_t)n_tile * NT * L);
        const int4* gs = reinterpret_cast<const int4*>(Bsmall + (int64_t)n_tile * NT * L);
        int4* db = reinterpret_cast<int4*>(sBb);
        int4* ds = reinterpret_cast<int4*>(sBs);
        for (int i = t; i < NT * L / 4; i += DEC_THREADS) {
            db[i] = __ldg(gb + i);
            ds[i] = __ldg(gs + i);
        }
    }
    if (t == 0) {
        for (int sidx = 0; sidx < 4; sidx++)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b_afree0 + 8 * sidx) : "memory");
        for (int sidx = 0; sidx < 2; sidx++) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b_full0 + 8 * sidx) : "memory");
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(b_empty0 + 8 * sidx), "r"(NUM_EPI) : "memory");
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp < NUM_PROD) {
        // ================= producers: A tile -> split -> smem; thread 0 issues the MMAs.
        // The tile is handled in KP parts along K (separate smem regions): part p of tile i+1 is
        // written as soon as the MMAs of part p of tile i are done, so splitting overlaps the
        // tensor-core work of the other part.
        constexpr int PT = NUM_PROD * 32;
        constexpr int KP = (L / 8) % 4 == 0 ? 4 : ((L / 8) % 2 == 0 ? 2 : 1);  // K parts
        constexpr int LP4 = L / 4 / KP;                // 16-byte chunks per row in a part
        constexpr int nqp = DM * LP4 / PT;             // chunks per producer thread per part
        constexpr int KS = L / 8 / KP;                 // k-steps (K = 8) per part
        const uint32_t idesc =
            (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(NT >> 3) << 17) | ((uint32_t)(DM >> 4) << 24);
        const uint32_t LBO = 128, SBO_A = (uint32_t)LP4 * 128, SBO_B = (uint32_t)(L / 4) * 128;
        const uint32_t bB = smem_u32(sBb), bS = smem_u32(sBs);
        // loop-invariant part of this thread's chunks.  In a part, chunk q lives at byte 16 q:
        // rows 8-grouped, (row % 8) fastest, then the k-chunk, then the group.
        int a_row[nqp], a_off[nqp];
#pragma unroll
        for (int j = 0; j < nqp; j++) {
            const int q = t + j * PT;
            const int rest = q >> 3, kc = rest % LP4;
            a_row[j] = (rest / LP4) * 8 + (q & 7);
            a_off[j] = a_row[j] * L + kc * 4;
        }
        float4 ra[KP][nqp];
        // part pp of tile mt into ra[pp]; issued right after part pp of the previous tile was
        // split, so each load has a whole tile period to land
        auto load_a = [&](int64_t mt, int pp) {
            if (mt >= mtiles) return;
            const float* At = A + mt * DM * L + pp * LP4 * 4;
            const int64_t left = P - 1 - mt * DM;
            const int lim = left < DM - 1 ? (int)left : DM - 1;  // last valid row of the tile
#pragma unroll
            for (int j = 0; j < nqp; j++) {
                // rows past P re-read the last valid row (zeroed at the split): no select on
                // the load result, so the loads stay in flight until the split
                const int off = a_row[j] <= lim ? a_off[j] : a_off[j] - (a_row[j] - lim) * L;
                ra[pp][j] = __ldg(reinterpret_cast<const float4*>(At + off));
            }
        };
#pragma unroll
        for (int pp = 0; pp < KP; pp++) load_a(m0, pp);
        int it = 0;
        for (int64_t m = m0; m < mtiles; m += mstep, it++) {
            const int st = it & 1;
#pragma unroll
            for (int pp = 0; pp < KP; pp++) {
                float* pAb = sAb + pp * DM * LP4 * 4;
                float* pAs = sAs + pp * DM * LP4 * 4;
                if (it > 0) mbar_wait(b_afree0 + 8 * pp, (uint32_t)(it - 1) & 1u);  // MMAs of this part done
#pragma unroll
                for (int j = 0; j < nqp; j++) {
                    const int q = t + j * PT;
                    const float4 x = m * DM + a_row[j] < P ? ra[pp][j] : make_float4(0.f, 0.f, 0.f, 0.f);
                    const float4 bg = make_float4(tf32_big(x.x), tf32_big(x.y), tf32_big(x.z), tf32_big(x.w));
                    reinterpret_cast<float4*>(pAb)[q] = bg;
                    reinterpret_cast<float4*>(pAs)[q] = make_float4(__fsub_rn(x.x, bg.x), __fsub_rn(x.y, bg.y),
                                                                    __fsub_rn(x.z, bg.z), __fsub_rn(x.w, bg.w));
                }
                load_a(m + mstep, pp);
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                asm volatile("bar.sync 1, %0;" ::"r"(PT) : "memory");
                if (t == 0) {
                    if (pp == 0 && it >= 2) mbar_wait(b_empty0 + 8 * st, (uint32_t)((it >> 1) - 1) & 1u);
                    fence_after();
                    const uint32_t dcol = tmem + (uint32_t)(st * 256);
                    const uint32_t aB = smem_u32(pAb), aS = smem_u32(pAs);
#pragma unroll
                    for (int k = 0; k < KS; k++) {
                        const uint32_t o = (uint32_t)k * 2 * LBO;  // K = 8 tf32 = two 16-byte chunks
                        const uint32_t ob = (uint32_t)(pp * KS + k) * 2 * LBO;
                        const uint64_t dab = umma_desc(aB + o, LBO, SBO_A), das = umma_desc(aS + o, LBO, SBO_A);
                        const uint64_t dbb = umma_desc(bB + ob, LBO, SBO_B), dbs = umma_desc(bS + ob, LBO, SBO_B);
                        mma_tf32(dcol, dab, dbb, idesc, (pp | k) > 0 ? 1u : 0u);
                        mma_tf32(dcol, dab, dbs, idesc, 1u);
                        mma_tf32(dcol, das, dbb, idesc, 1u);
                    }
                    if (pp == KP - 1)
                        asm volatile(
                            "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                                b_full0 + 8 * st)
                            : "memory");
                    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                                     b_afree0 + 8 * pp)
                                 : "memory");
                }
                __syncwarp();
            }
        }
    } else {
        // ================= epilogue: TMEM -> registers -> swizzled staging -> TMA store to F
        const int e = warp - NUM_PROD;
        const int qw = warp & 3, ch = e >> 2;  // TMEM lane quarter (hardware: warp id mod 4), column part
        const int span = NT * 4 / NUM_EPI;    // columns per epilogue warp
        float* stg = stg_base + e * NB * 1024;  // NB 32 x 32 fp32 blocks
        const int col0 = n_tile * NT + ch * span;
        int nstore = 0;
        // one 32-row x 32-column block: row = lane, 16-byte chunk u at u ^ (row % 8) (the TMA
        // 128-byte swizzle, which also makes these stores bank-conflict free), then one thread
        // hands the block to the TMA engine (rows past P are clipped by the tensor map)
        auto drain = [&](const uint32_t(&v)[32], int64_t row0, int c0) {
            float* buf = stg + (nstore % NB) * 1024;
            if (nstore >= NB) {
                if (lane == 0) asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(NB - 1) : "memory");
                __syncwarp();
            }
#pragma unroll
            for (int u = 0; u < 8; u++)
                *reinterpret_cast<uint4*>(buf + lane * 32 + ((u ^ (lane & 7)) << 2)) =
                    make_uint4(v[4 * u], v[4 * u + 1], v[4 * u + 2], v[4 * u + 3]);
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            if (lane == 0) {
                asm volatile(
                    "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                        reinterpret_cast<uint64_t>(&tmap_F)),
                    "r"(col0 + c0), "r"((int)row0), "r"(smem_u32(buf))
                    : "memory");
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            }
            nstore++;
        };
        int it = 0;
        for (int64_t m = m0; m < mtiles; m += mstep, it++) {
            const int st = it & 1;
            mbar_wait(b_full0 + 8 * st, (uint32_t)(it >> 1) & 1u);
            fence_after();
            const int64_t row0 = m * DM + qw * 32;
            const uint32_t tbase = tmem + ((uint32_t)(qw * 32) << 16) + (uint32_t)(st * 256 + ch * span);
            for (int c0 = 0; c0 < span; c0 += 64) {  // span is a multiple of 32; two loads in flight
                uint32_t v0[32], v1[32];
                tmem_ld32(tbase + c0, v0);
                if (c0 + 32 < span) tmem_ld32(tbase + c0 + 32, v1);
                tmem_wait_ld();
                drain(v0, row0, c0);
                if (c0 + 32 < span) drain(v1, row0, c0 + 32);
            }
            fence_before();
            __syncwarp();
            if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(b_empty0 + 8 * st) : "memory");
        }
        if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
        __syncwarp();
    }
    fence_before();
    __syncthreads();
    fence_after();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
}

}  // namespace

bool decode_tc_supported(int L, int D) { return L >= 8 && L <= 64 && L % 8 == 0 && D >= 64 && D % 64 == 0; }

#ifndef DEC_NTMAX
#define DEC_NTMAX 256
#endif
static int decode_nt(int D) { return (D % 256 == 0 && DEC_NTMAX >= 256) ? 256 : (D % 128 == 0 ? 128 : 64); }

size_t decode_tc_scratch_bytes(int L, int D) { return 2 * sizeof(float) * (size_t)L * D; }

cudaError_t launch_decode_tc(const float* W_hat, int64_t P, int L, int D, const float* C, float* scratch, float* F,
                             int num_sms, cudaStream_t s) {
    const int NT = decode_nt(D);
    float* Bbig = scratch;
    float* Bsmall = scratch + (size_t)L * D;
    decode_prep_kernel<<<(L * D + 255) / 256, 256, 0, s>>>(C, L, D, NT, Bbig, Bsmall);
    // F [P, D] as a 2-D tensor for the TMA stores: 32 x 32 fp32 boxes, 128-byte swizzle
    static PFN_cuTensorMapEncodeTiled encode = nullptr;
    if (!encode) {
        cudaDriverEntryPointQueryResult q{};
        void* fn = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn)
            return cudaErrorNotSupported;
        encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled>(fn);
    }
    CUtensorMap tmap;
    const cuuint64_t gdim[2] = {(cuuint64_t)D, (cuuint64_t)P};
    const cuuint64_t gstride[1] = {(cuuint64_t)D * sizeof(float)};
    const cuuint32_t box[2] = {32, 32}, estride[2] = {1, 1};
    if (encode(&tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, F, gdim, gstride, box, estride, CU_TENSOR_MAP_INTERLEAVE_NONE,
               CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return cudaErrorInvalidValue;
    const int nN = D / NT;
    const size_t smem = sizeof(float) * (size_t)(2 * NT * L + 2 * DM * L + NUM_EPI * NB * 1024) + 128;
    const int64_t mtiles = (P + DM - 1) / DM;
    int64_t per = std::max(1, num_sms / nN);
    per = std::min<int64_t>(per, mtiles);
    auto go = [&](auto kern) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        kern<<<(unsigned)(per * nN), DEC_THREADS, smem, s>>>(W_hat, P, D, NT, Bbig, Bsmall, tmap);
    };
    switch (L) {
        case 8: go(decode_kernel<8>); break;
        case 16: go(decode_kernel<16>); break;
        case 24: go(decode_kernel<24>); break;
        case 32: go(decode_kernel<32>); break;
        case 40: go(decode_kernel<40>); break;
        case 48: go(decode_kernel<48>); break;
        case 56: go(decode_kernel<56>); break;
        default: go(decode_kernel<64>); break;
    }
    return cudaGetLastError();
}

}  // namespace scoup
