// raster2.cu -- the fused rasterise-and-aggregate kernel with TWO pixels per thread: the
// production path of the single-level sparse uplift (every BASELINE config; Algorithm 1
// lines 5-12).  Multi-level passes and dense features keep raster.cu's kernel.
//
// One CTA of 128 threads (4 warps) per (view, 16x16 tile); warp w covers the 8x8 block at
// column 8*(w&1), row 8*(w>>1) of the tile; lane l owns pixels (x, yA) and (x, yA + 4) with
// x = 8*(w&1) + (l&7), yA = 8*(w>>1) + (l>>3).  The tile walks its bin's depth-ordered list:
//
//  refill   128 candidates per round (records fetched one round ahead with cp.async), tested
//           against the tile (band_relevant, conservative) and stably compacted into a ring;
//  batch    up to 2 sub-batches of 32 ring records per barrier; per sub-batch each warp ballots
//           the records that may touch its 8x8 block, and per group of 8 records (one warp-
//           uniform branch) every lane evaluates DESIGN.md §3 step PX for its TWO pixels: the
//           record's scalars (dx, the square test on x, the loads) are shared, and everything
//           per pixel -- dy, the quadratic form, exp2_spec, o 2^q, 1 - alpha, the transmittance
//           T(1 - alpha) and the weight alpha T -- runs in paired FP32 (FADD2 / FMUL2 / FFMA2,
//           each half an IEEE round-to-nearest op, so every e_i(v,p) of PAPER.md Eq. 2 is
//           bit-identical to the oracle's);
//  reduce   after each group: the 8 records' weights, summed over the lane's two pixels when
//           they share a region slot, are reduced over the warp by an 8-value transpose-
//           reduction (7 exchanges + 2 xor-adds) and added to per-(slot, record) shared sums;
//  flush    after the barrier: S `red.global.add.f32` per (slot, Gaussian) into W[g][atom]
//           (c * sum e, Eq. 5) and one per Gaussian into Z[g] (sum over slots).
//
// The per-thread transmittance uses the "dead below 1e-4" convention of raster.cu (a pixel is
// finished once T < 1e-4; DESIGN.md §4 R9).
#include <algorithm>
#include <cstdlib>

#include "internal.cuh"

namespace scoup {

namespace {

constexpr unsigned FULL = 0xffffffffu;
constexpr uint32_t KEY_NONE = 0xFFFFFFFFu;   // unassigned or outside the image
constexpr uint32_t SLOT_EMPTY = 0xFFFFFFFEu;  // slot-table sentinel
constexpr int R2T = 128;                      // threads per CTA (4 warps, 2 pixels each)
constexpr int R2W = R2T / 32;
#ifndef RASTER2_RING
#define RASTER2_RING 192                      // ring capacity (>= 63 + 128 records in flight; a multiple of 32)
#endif
constexpr int R2Q = RASTER2_RING;
#ifndef RASTER2_NSUB
#define RASTER2_NSUB 2                        // sub-batches of BATCH records per barrier
#endif
#ifndef RASTER2_SLOTS
#define RASTER2_SLOTS 8                       // distinct regions per tile on the shared-sum path (more: per-pixel path)
#endif
#ifndef RASTER2_SLOTS_FEW
#define RASTER2_SLOTS_FEW 4                   // ... of the small-footprint variant for views with large regions
#endif
constexpr int R2SB = RASTER2_NSUB * BATCH;    // records per super-batch (one barrier, one flush)
constexpr int RG = 8;                         // records per warp-uniform group (and per reduction)
#ifndef RASTER2_FLUSH_SPLIT
#define RASTER2_FLUSH_SPLIT 2                 // threads per (slot, record) in the flush (a power of two)
#endif
constexpr int R2FS = RASTER2_FLUSH_SPLIT;
#ifndef RASTER2_MIN_BLOCKS
#define RASTER2_MIN_BLOCKS 7
#endif

static_assert(BATCH == 32 && (R2SB & (R2SB - 1)) == 0 && R2SB <= R2T, "sub-batches of one record per lane");
static_assert(RASTER2_SLOTS <= MAX_SLOTS && RASTER2_SLOTS_FEW <= RASTER2_SLOTS, "slot table");
static_assert(R2Q >= R2SB - 1 + R2T && R2Q % BATCH == 0, "ring holds a round on top of a partial super-batch");
// ring position of x < 2 R2Q (every use: head < R2Q plus less than R2SB + R2T)
__device__ __forceinline__ uint32_t ring_wrap(uint32_t x) {
    if ((R2Q & (R2Q - 1)) == 0) return x & (uint32_t)(R2Q - 1);
    return x >= (uint32_t)R2Q ? x - (uint32_t)R2Q : x;
}

template <int R2S>
struct __align__(16) R2Smem {
    float4 rp[R2Q];   // (mx, my, r, o)
    float4 rq[R2Q];   // (qa, qb, qc, ycut)
    float4 re[R2Q];   // (support-box half-extents x, y, Gaussian id bits, sy)
    float4 rb[R2Q];   // band_relevant parameters
    // per (slot, record) sums of a super-batch, triple-buffered as in raster.cu: each warp's
    // primary slot (its lowest) in its own row accw (plain stores -- sm_100 has no native
    // shared-memory FP32 atomic add, atomicAdd there is a CAS loop), its other slots in acc
    // (CAS atomics; warps with more than one slot are the minority)
    float acc[3][R2S * R2SB];
    float accw[3][R2W][R2SB];
    int wslot[R2W];
    float4 st0[R2T], st1[R2T], st2[R2T], st3[R2T];  // next round's candidates (cp.async staging)
    uint32_t slot_key[R2S];
    uint32_t slot_atom[R2S][MAX_S];
    float slot_coef[R2S][MAX_S];
    int nslot;
    int overflow;
    int wcnt[2][R2W];  // accepted candidates per warp, double-buffered over refill rounds
    unsigned long long contrib, tests, evals, reds;
#ifdef RASTER2_PAD
    unsigned char pad[RASTER2_PAD];  // (A/B: residency limited by shared memory at a given register count)
#endif
};

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool pred) {
    const uint32_t sa = (uint32_t)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(gmem), "r"(pred ? 16 : 0));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }

// Sum v[0..7] over the 32 lanes; lane l returns the sum for record l & 7.  Butterfly over lane
// bits 2, 1, 0 (each lane keeps the half of the records its bit selects), then the four 8-lane
// groups are added (xor 8, xor 16).
__device__ __forceinline__ float transpose8(float (&v)[RG], int lane) {
    {
        const bool up = lane & 4;
#pragma unroll
        for (int i = 0; i < 4; i += 2) {
            const float s0 = __shfl_xor_sync(FULL, up ? v[i] : v[i + 4], 4);
            const float s1 = __shfl_xor_sync(FULL, up ? v[i + 1] : v[i + 5], 4);
            f2_split(f2_add(f2_pack(up ? v[i + 4] : v[i], up ? v[i + 5] : v[i + 1]), f2_pack(s0, s1)), v[i], v[i + 1]);
        }
    }
    {
        const bool up = lane & 2;
        const float s0 = __shfl_xor_sync(FULL, up ? v[0] : v[2], 2);
        const float s1 = __shfl_xor_sync(FULL, up ? v[1] : v[3], 2);
        f2_split(f2_add(f2_pack(up ? v[2] : v[0], up ? v[3] : v[1]), f2_pack(s0, s1)), v[0], v[1]);
    }
    {
        const bool up = lane & 1;
        v[0] = (up ? v[1] : v[0]) + __shfl_xor_sync(FULL, up ? v[0] : v[1], 1);
    }
    float r = v[0];
    r += __shfl_xor_sync(FULL, r, 8);
    r += __shfl_xor_sync(FULL, r, 16);
    return r;
}

// alpha if the fragment passes the §3 PX tests (live, |dx| <= r, |dy| <= r, !(q > 0), the
// conservative q >= ycut, alpha >= 1/255), else 0 -- one predicate chain, one select.
__device__ __forceinline__ float pass_select(float al, float adx, float ady, float r, float q, float ycut,
                                             uint32_t live) {
    float out;
    asm("{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %7, 0;\n\t"
        "setp.le.and.f32 p, %2, %4, p;\n\t"
        "setp.le.and.f32 p, %3, %4, p;\n\t"
        "setp.leu.and.f32 p, %5, 0f00000000, p;\n\t"
        "setp.ge.and.f32 p, %5, %6, p;\n\t"
        "setp.ge.and.f32 p, %1, 0f3B808081, p;\n\t"
        "selp.f32 %0, %1, 0f00000000, p;\n\t}"
        : "=f"(out)
        : "f"(al), "f"(adx), "f"(ady), "f"(r), "f"(q), "f"(ycut), "r"(live));
    return out;
}

// Fallback aggregation of one fragment (tiles with > MAX_SLOTS regions): the pixel's code and Z.
__device__ __noinline__ void overflow_red1(float* W, float* Z, const uint32_t* atoms, const float* coefs, int S, int L,
                                           uint32_t g, float ev, int64_t row) {
    atomicAdd(Z + g, ev);
    if (row < 0) return;
    for (int s = 0; s < S; s++) {
        const uint32_t at = __ldg(atoms + row + s);
        if (at != NONE) atomicAdd(W + (int64_t)g * L + at, __fmul_rn(__ldg(coefs + row + s), ev));
    }
}

template <bool COUNT, int R2S>
__global__ void __launch_bounds__(R2T, RASTER2_MIN_BLOCKS) raster2_kernel(const RasterParams p) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    R2Smem<R2S>& sm = *reinterpret_cast<R2Smem<R2S>*>(smem_raw);
    const int ntiles = p.bn.tiles_x * p.bn.tiles_y;
    const int view = blockIdx.x / ntiles, tile = blockIdx.x - view * ntiles;
    const int tx = tile % p.bn.tiles_x, ty = tile / p.bn.tiles_x;
    const int64_t gtile = (int64_t)view * ntiles + tile;
    if (p.chunk > 0 && !p.tile_live[gtile]) return;  // every pixel finished in an earlier chunk
    const int bin = ((ty * TILE) >> p.bn.bshy) * p.bn.bins_x + ((tx * TILE) >> p.bn.bshx);
    const uint2 range = p.ranges[view * p.bn.nbins() + bin];
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const int wx0 = tx * TILE + 8 * (warp & 1), wy0 = ty * TILE + 8 * (warp >> 1);
    const int x = wx0 + (lane & 7), yA = wy0 + (lane >> 3), yB = yA + 4;
    const int Wd = p.width, Hd = p.height;
    const bool inA = x < Wd && yA < Hd, inB = x < Wd && yB < Hd;
    float* const TpA = p.Tstate + (int64_t)view * Wd * Hd + (int64_t)yA * Wd + x;
    float* const TpB = TpA + 4 * (int64_t)Wd;
    if (range.x >= range.y) {  // nothing of this chunk reaches the tile
        if (p.chunk == 0) {
            if (inA) *TpA = 1.0f;
            if (inB) *TpB = 1.0f;
            if (t == 0) p.tile_live[gtile] = 1;
        }
        return;
    }
    // software-pipelined candidate fetch (one candidate per thread per round), issued before the
    // slot setup so its two dependent global latencies overlap the region-id and code loads
    auto prefetch = [&](uint32_t e, bool ok) {
        const uint32_t es = ok ? e : 0u;
        cp_async16(&sm.st0[t], p.rec0 + es, ok);
        cp_async16(&sm.st1[t], p.rec1 + es, ok);
        cp_async16(&sm.st2[t], p.rec2 + es, ok);
        cp_async16(&sm.st3[t], p.rec3 + es, ok);
        cp_async_commit();
    };
    uint32_t cursor = range.x;
    {
        const bool ok = cursor + t < range.y;
        prefetch(ok ? __ldg(p.eval + cursor + t) : 0u, ok);
    }
    uint32_t e_next = cursor + R2T + t < range.y ? __ldg(p.eval + cursor + R2T + t) : 0u;

    // pixel-centre rectangles of the tile and of this warp's 8x8 block (clipped to the image)
    const float TX0 = (float)(tx * TILE) + 0.5f, TY0 = (float)(ty * TILE) + 0.5f;
    const float TX1 = (float)(min(tx * TILE + TILE, Wd) - 1) + 0.5f;
    const float TY1 = (float)(min(ty * TILE + TILE, Hd) - 1) + 0.5f;
    const float WX0 = (float)wx0 + 0.5f, WY0 = (float)wy0 + 0.5f;
    const float WX1 = (float)(min(wx0 + 8, Wd) - 1) + 0.5f, WY1 = (float)(min(wy0 + 8, Hd) - 1) + 0.5f;

    // ---- setup: region ids of my two pixels, the tile's slot table, slot codes
    auto region = [&](bool in, int yy) {
        uint32_t rid = KEY_NONE;
        if (in) {
            rid = __ldg(p.region_ids[view][0] + (int64_t)yy * Wd + x);
            if (rid != NONE && rid >= (uint32_t)p.num_regions[view][0]) {
                latch_error(p.err, ERR_REGION, p.pixel_base[view] + (int64_t)yy * Wd + x);
                rid = NONE;
            }
        }
        return rid;
    };
    const uint32_t kA = region(inA, yA), kB = region(inB, yB);
    if (t == 0) { sm.nslot = 0; sm.overflow = 0; sm.contrib = 0ull; sm.tests = 0ull; sm.evals = 0ull; sm.reds = 0ull; }
    if (t < R2S) sm.slot_key[t] = SLOT_EMPTY;
    for (int i = t; i < 3 * R2S * R2SB; i += R2T) (&sm.acc[0][0])[i] = 0.f;
    for (int i = t; i < 3 * R2W * R2SB; i += R2T) (&sm.accw[0][0][0])[i] = 0.f;
    __syncthreads();
    // one claim per distinct key per warp (CAS: the first empty or matching slot)
    auto claim = [&](uint32_t k) {
        const unsigned g = __match_any_sync(FULL, k);
        const int leader = __ffs(g) - 1;
        int sl = -1;
        if (lane == leader) {
            for (int q = 0; q < R2S; q++) {
                const uint32_t old = atomicCAS(&sm.slot_key[q], SLOT_EMPTY, k);
                if (old == SLOT_EMPTY || old == k) { sl = q; break; }
            }
            if (sl < 0) sm.overflow = 1;
            else atomicMax(&sm.nslot, sl + 1);
        }
        return __shfl_sync(FULL, sl, leader);
    };
    const int slA = max(0, claim(kA)), slB = max(0, claim(kB));
    __syncthreads();
    const int nslot = sm.nslot;
    const bool overflow = sm.overflow != 0;
    const int S = p.S, L = p.L;
    const int s_log2 = (S & (S - 1)) == 0 ? __ffs(S) - 1 : -1;
    const uint32_t s_magic = 0xFFFFFFFFu / (uint32_t)S + 1u;  // ceil(2^32 / S): i / S by multiply-high
    for (int i = t; i < nslot * S; i += R2T) {
        const int q = s_log2 >= 0 ? i >> s_log2 : (int)__umulhi((uint32_t)i, s_magic);
        const int s = i - q * S;
        const uint32_t k = sm.slot_key[q];
        uint32_t a = NONE;
        float c = 0.f;
        if (k != KEY_NONE) {
            const int64_t row = (p.code_row0[view][0] + (int64_t)k) * S + s;
            a = __ldg(p.code_atoms + row);
            c = __ldg(p.code_coefs + row);
        }
        sm.slot_atom[q][s] = a;
        sm.slot_coef[q][s] = c;
    }
    // the warp's slots (bit q: some pixel of the warp is in slot q); one slot for both pixels of
    // every lane -- the common case -- sums the two pixels' weights before the reduction
    const unsigned wslots = __reduce_or_sync(FULL, (1u << slA) | (1u << slB));
    const bool one_slot = (wslots & (wslots - 1)) == 0;
    const int slot0 = __ffs(wslots) - 1;  // the warp's primary slot
    if (lane == 0) sm.wslot[warp] = slot0;

    const float px = __fadd_rn((float)x, 0.5f);
    const f2 PY = f2_pack(__fadd_rn((float)yA, 0.5f), __fadd_rn((float)yB, 0.5f));
    // transmittance of both pixels; T < 1e-4: finished (0 outside the image)
    float TA = !inA ? 0.0f : (p.chunk == 0 ? 1.0f : *TpA);
    float TB = !inB ? 0.0f : (p.chunk == 0 ? 1.0f : *TpB);
    uint32_t cnt = 0, tests = 0, wevals = 0, nred = 0;
    const unsigned lanemask_lt = (1u << lane) - 1u;
    uint32_t q_head = 0, q_count = 0;
    int buf = 0, rbuf = 0;
    while (true) {
        // ---- refill the ring (stable compaction of the round's accepted candidates).  One
        // barrier per round (the per-warp counts are double-buffered, so the next round's counts
        // never overwrite ones still being read) and one after the last round's ring writes.
        bool refilled = false;
        while (q_count < (uint32_t)R2SB && cursor < range.y) {
            const uint32_t idx = cursor + t;
            cp_async_wait_all();
            const float4 r0 = sm.st0[t], r1 = sm.st1[t], r2 = sm.st2[t], r3 = sm.st3[t];
            const bool acc = idx < range.y && band_relevant(r0, r2, r3, TX0, TX1, TY0, TY1);
            {
                const uint32_t nidx = cursor + R2T + t;
                prefetch(e_next, nidx < range.y);
                e_next = nidx + R2T < range.y ? __ldg(p.eval + nidx + R2T) : 0u;
            }
            const unsigned bal = __ballot_sync(FULL, acc);
            if (lane == 0) sm.wcnt[rbuf][warp] = __popc(bal);
            __syncthreads();
            uint32_t off = 0, tot = 0;
#pragma unroll
            for (int w = 0; w < R2W; w++) {
                const uint32_t c = (uint32_t)sm.wcnt[rbuf][w];
                off += (w < warp) ? c : 0u;
                tot += c;
            }
            if (acc) {
                const uint32_t pos = ring_wrap(q_head + q_count + off + __popc(bal & lanemask_lt));
                sm.rp[pos] = r0;
                sm.rq[pos] = r1;
                sm.re[pos] = r2;
                sm.rb[pos] = r3;
            }
            q_count += tot;
            cursor += R2T;
            rbuf ^= 1;
            refilled = true;
        }
        if (refilled) __syncthreads();
        if (q_count == 0) break;
        const uint32_t n = min((uint32_t)R2SB, q_count);
        const int nsub = (int)((n + BATCH - 1) / BATCH);
        if (n % BATCH) {
            // the tile's last, partial sub-batch: blank the stale ring slots after it (a negative
            // support radius fails every square test)
            if ((uint32_t)t >= n && t < nsub * BATCH) sm.rp[ring_wrap(q_head + (uint32_t)t)].z = -1.0f;
            __syncthreads();
        }
#pragma unroll 1
        for (int sb = 0; sb < nsub; sb++) {
            const uint32_t sh = ring_wrap(q_head + (uint32_t)(sb * BATCH));  // contiguous: sh % 32 == 0
            const uint32_t nsb = min((uint32_t)BATCH, n - (uint32_t)(sb * BATCH));
            const bool warp_done = __all_sync(FULL, !(TA >= K_TMIN) && !(TB >= K_TMIN));
            bool rel = false;
            if (!warp_done && (uint32_t)lane < nsb)
                rel = band_relevant(sm.rp[sh + lane], sm.re[sh + lane], sm.rb[sh + lane], WX0, WX1, WY0, WY1);
            const unsigned mask = __ballot_sync(FULL, rel);
            const float4* const RP = sm.rp + sh;
            const float4* const RQ = sm.rq + sh;
            // (the group loop stays rolled: one copy of the group body keeps the kernel's code
            // within the instruction cache)
#pragma unroll 1
            for (int g0 = 0; g0 < BATCH; g0 += RG) {
                if (!((mask >> g0) & ((1u << RG) - 1u))) continue;  // warp-uniform
                float eA[RG], eB[RG];
#pragma unroll
                for (int jj = 0; jj < RG; jj++) {
                    // DESIGN.md §3 PX for record g0 + jj at both pixels: the record's scalars
                    // once, the per-pixel chain in paired FP32 (each half the scalar IEEE op)
                    const float4 a = RP[g0 + jj], b = RQ[g0 + jj];
                    const float dx = __fsub_rn(px, a.x);
                    const f2 DX = f2_pack(dx, dx);
                    const f2 dy = f2_sub(PY, f2_pack(a.y, a.y));                       // py - my
                    const f2 q = f2_fma(DX, f2_fma(f2_pack(b.x, b.x), DX, f2_mul(f2_pack(b.y, b.y), dy)),
                                        f2_mul(f2_mul(f2_pack(b.z, b.z), dy), dy));
                    const f2 ex = exp2_spec2(q);
                    float mA, mB;
                    f2_split(f2_mul(f2_pack(a.w, a.w), ex), mA, mB);                   // o * exp2_spec(q)
                    float dyA, dyB, qA, qB;
                    f2_split(dy, dyA, dyB);
                    f2_split(q, qA, qB);
                    const bool sqx = (!COUNT || ((mask >> (g0 + jj)) & 1u)) && fabsf(dx) <= a.z;
                    const bool sqA = sqx && fabsf(dyA) <= a.z, sqB = sqx && fabsf(dyB) <= a.z;
                    float alA = fminf(K_ACLAMP, mA), alB = fminf(K_ACLAMP, mB);
                    const bool passA = sqA && !(qA > 0.f) && qA >= b.w && alA >= K_AMIN;
                    const bool passB = sqB && !(qB > 0.f) && qB >= b.w && alB >= K_AMIN;
                    // a fragment that does not pass takes alpha = 0: T (1 - 0) = T exactly and
                    // alpha T = 0, so T needs no select (pass && Tn < 1e-4: the pixel ends).  The
                    // pass test as one predicate chain per pixel and a single select (PTX: the
                    // compiler otherwise splits the && chain into one select per condition)
                    alA = pass_select(alA, fabsf(dx), fabsf(dyA), a.z, qA, b.w, COUNT ? ((mask >> (g0 + jj)) & 1u) : 1u);
                    alB = pass_select(alB, fabsf(dx), fabsf(dyB), a.z, qB, b.w, COUNT ? ((mask >> (g0 + jj)) & 1u) : 1u);
                    const f2 AL = f2_pack(alA, alB);
                    const f2 T2 = f2_pack(TA, TB);
                    float TnA, TnB, wA, wB;
                    f2_split(f2_mul(T2, f2_rsub(AL, 1.0f)), TnA, TnB);                 // T (1 - alpha)
                    f2_split(f2_mul(AL, T2), wA, wB);                                   // alpha T
                    if (COUNT) {
                        const bool conA = passA && !(TnA < K_TMIN), conB = passB && !(TnB < K_TMIN);
                        cnt += (conA ? 1u : 0u) + (conB ? 1u : 0u);
                        tests += ((sqA && TA >= K_TMIN) ? 1u : 0u) + ((sqB && TB >= K_TMIN) ? 1u : 0u);
                    }
                    // e = w where the pixel continues (!(Tn < 1e-4)), else 0 (w = 0 unless the
                    // fragment passes): w times a 1.0 / 0.0 flag (PTX set: one ALU op per pixel
                    // instead of a compare and a select; the product is exact)
                    float gA, gB;
                    asm("set.geu.f32.f32 %0, %1, %2;" : "=f"(gA) : "f"(TnA), "f"(K_TMIN));
                    asm("set.geu.f32.f32 %0, %1, %2;" : "=f"(gB) : "f"(TnB), "f"(K_TMIN));
                    f2_split(f2_mul(f2_pack(wA, wB), f2_pack(gA, gB)), eA[jj], eB[jj]);
                    TA = TnA;
                    TB = TnB;
                }
                if (COUNT) wevals += 2 * RG;
                // ---- reduce the group's weights per (slot, record) into the shared sums
                const int col = sb * BATCH + g0;
                if (!overflow) {
                    if (one_slot) {
                        float v[RG];
#pragma unroll
                        for (int jj = 0; jj < RG; jj++) v[jj] = eA[jj] + eB[jj];
                        const float s = transpose8(v, lane);
                        if (lane < RG) sm.accw[buf][warp][col + lane] = s;
                    } else {
                        unsigned todo = wslots;
                        while (todo) {
                            const int q = __ffs(todo) - 1;
                            todo &= todo - 1;
                            float v[RG];
#pragma unroll
                            for (int jj = 0; jj < RG; jj++) v[jj] = (slA == q ? eA[jj] : 0.f) + (slB == q ? eB[jj] : 0.f);
                            const float s = transpose8(v, lane);
                            if (lane < RG) {
                                if (q == slot0) sm.accw[buf][warp][col + lane] = s;
                                else if (s != 0.f) atomicAdd(&sm.acc[buf][q * R2SB + col + lane], s);
                            }
                        }
                    }
                } else {
                    // > MAX_SLOTS regions in the tile: per-pixel reductions from the code table
#pragma unroll
                    for (int jj = 0; jj < RG; jj++) {
                        const uint32_t gid = __float_as_uint(sm.re[sh + g0 + jj].z);
                        if (eA[jj] > 0.f)
                            overflow_red1(p.W, p.Z, p.code_atoms, p.code_coefs, S, L, gid, eA[jj],
                                          kA != NONE && kA != KEY_NONE ? (p.code_row0[view][0] + (int64_t)kA) * S : -1);
                        if (eB[jj] > 0.f)
                            overflow_red1(p.W, p.Z, p.code_atoms, p.code_coefs, S, L, gid, eB[jj],
                                          kB != NONE && kB != KEY_NONE ? (p.code_row0[view][0] + (int64_t)kB) * S : -1);
                    }
                }
            }
        }
        // the super-batch's sums are complete; termination vote (all pixels finished)
        const int alive = __syncthreads_count(TA >= K_TMIN || TB >= K_TMIN);
        if (!overflow) {
            int ws[R2W];  // the warps' primary slots (their sums are in accw)
#pragma unroll
            for (int w = 0; w < R2W; w++) ws[w] = sm.wslot[w];
            // ---- flush: S reds per (slot, record) into W, one per record into Z (sum over slots)
            const int ncol = nsub * BATCH;
            auto gid_of = [&](int j) { return __float_as_uint(sm.re[ring_wrap(q_head + (uint32_t)j)].z); };
            // R2FS threads per (slot, record): the pair's sum once per thread, then the thread's
            // share of the S atoms (s = i mod R2FS, + R2FS, ...)
            const int nitems = nslot * R2SB * R2FS;
            for (int i = t; i < nitems; i += R2T) {
                const int u = i / R2FS;  // (slot, record)
                const int j = u & (R2SB - 1), q = u / R2SB;
                if (j >= ncol) continue;
                float v = sm.acc[buf][u];
#pragma unroll
                for (int w = 0; w < R2W; w++)
                    if (ws[w] == q) v += sm.accw[buf][w][j];
                if (v > 0.f) {
                    float* const Wg = p.W + (int64_t)gid_of(j) * L;
                    for (int s = i & (R2FS - 1); s < S; s += R2FS) {
                        const uint32_t a = sm.slot_atom[q][s];
                        if (a != NONE) {
                            if (COUNT) nred++;
                            atomicAdd(Wg + a, __fmul_rn(sm.slot_coef[q][s], v));
                        }
                    }
                }
            }
            if (t < ncol) {
                float z = 0.f;
                for (int q = 0; q < nslot; q++) z += sm.acc[buf][q * R2SB + t];
#pragma unroll
                for (int w = 0; w < R2W; w++) z += sm.accw[buf][w][t];
                if (z > 0.f) {
                    if (COUNT) nred++;
                    atomicAdd(p.Z + gid_of(t), z);
                }
            }
            // zero the buffer of super-batch i+2 (flushed in super-batch i-1, before this barrier)
            const int bz = buf == 0 ? 2 : buf - 1;
            for (int i = t; i < nslot * R2SB; i += R2T) sm.acc[bz][i] = 0.f;
            for (int i = t; i < R2W * R2SB; i += R2T) (&sm.accw[bz][0][0])[i] = 0.f;
        }
        q_head = ring_wrap(q_head + n);
        q_count -= n;
        buf = buf == 2 ? 0 : buf + 1;
        if (alive == 0) break;
    }

    cp_async_wait_all();  // no copy may land in shared memory after the CTA retires

    // carry the per-pixel state to the next chunk
    if (inA) *TpA = TA;
    if (inB) *TpB = TB;
    const int live = __syncthreads_count(TA >= K_TMIN || TB >= K_TMIN);
    if (t == 0) p.tile_live[gtile] = live > 0 ? 1 : 0;

    if (COUNT) {
        const unsigned c = __reduce_add_sync(FULL, cnt), ts = __reduce_add_sync(FULL, tests),
                       rs = __reduce_add_sync(FULL, nred);
        if (lane == 0) {
            if (c) atomicAdd(&sm.contrib, (unsigned long long)c);
            if (ts) atomicAdd(&sm.tests, (unsigned long long)ts);
            if (wevals) atomicAdd(&sm.evals, 32ull * wevals);
            if (rs) atomicAdd(&sm.reds, (unsigned long long)rs);
        }
        __syncthreads();
        if (t == 0) {
            if (sm.contrib) {
                atomicAdd(p.contrib_ctr, sm.contrib);
                if (p.contrib_out[view]) atomicAdd(reinterpret_cast<unsigned long long*>(p.contrib_out[view]), sm.contrib);
            }
            if (sm.tests) atomicAdd(p.support_ctr, sm.tests);
            if (sm.evals) atomicAdd(p.lane_eval_ctr, sm.evals);
            if (sm.reds) atomicAdd(p.red_ctr, sm.reds);
        }
    }
}

}  // namespace

bool raster2_supported(const RasterParams& p) {
    return p.nlev == 1 && !p.dense && p.S <= MAX_S;
}

// Slots per tile.  The variant with RASTER2_SLOTS_FEW slots has the smaller shared-memory
// footprint (27.9 KB against 30.9 KB per CTA: the front kernels of the other pipeline context fit
// next to 7 resident raster CTAs sooner, measured -2 ms per outdoor step); it serves batches
// whose regions average at least 64 x 64 px (4 x 4 tiles: a tile then rarely meets more than 4
// regions -- tiles that do take the per-pixel path in either variant).  SCOUP_RASTER2_SLOTS
// or scoup_diag_set_raster2_slots (4 or 8) forces one variant.
static int g_slots_override = -1;  // scoup_diag_set_raster2_slots (-1: SCOUP_RASTER2_SLOTS, else adaptive)

static int raster2_slots(const RasterParams& p) {
    if (g_slots_override < 0) {
        const char* e = getenv("SCOUP_RASTER2_SLOTS");
        g_slots_override = e ? std::max(0, atoi(e)) : 0;
    }
    if (g_slots_override > 0) return g_slots_override <= RASTER2_SLOTS_FEW ? RASTER2_SLOTS_FEW : RASTER2_SLOTS;
    const int64_t area = (int64_t)p.width * p.height;
    for (int v = 0; v < p.nviews; v++)
        if ((int64_t)p.num_regions[v][0] * 4096 > area) return RASTER2_SLOTS;
    return RASTER2_SLOTS_FEW;
}

template <int R2S>
static void launch_raster2_slots(const RasterParams& p, int nblocks, cudaStream_t s) {
#ifndef RASTER2_PAD
    static_assert(RASTER2_MIN_BLOCKS * (sizeof(R2Smem<R2S>) + 1024) <= 228 * 1024, "shared memory per SM");
#endif
    static bool attr_set = false;
    if (!attr_set) {
        cudaFuncSetAttribute(raster2_kernel<true, R2S>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)sizeof(R2Smem<R2S>));
        cudaFuncSetAttribute(raster2_kernel<false, R2S>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)sizeof(R2Smem<R2S>));
        if (const char* e = getenv("SCOUP_RASTER2_CARVEOUT")) {  // (A/B) percent of the L1 / shared array
            cudaFuncSetAttribute(raster2_kernel<true, R2S>, cudaFuncAttributePreferredSharedMemoryCarveout, atoi(e));
            cudaFuncSetAttribute(raster2_kernel<false, R2S>, cudaFuncAttributePreferredSharedMemoryCarveout, atoi(e));
        }
        attr_set = true;
    }
    if (p.count_tests) raster2_kernel<true, R2S><<<nblocks, R2T, sizeof(R2Smem<R2S>), s>>>(p);
    else raster2_kernel<false, R2S><<<nblocks, R2T, sizeof(R2Smem<R2S>), s>>>(p);
}

void launch_raster2(const RasterParams& p, cudaStream_t s) {
    const int nblocks = p.bn.tiles_x * p.bn.tiles_y * p.nviews;
    if (nblocks <= 0) return;
    if (raster2_slots(p) == RASTER2_SLOTS_FEW) launch_raster2_slots<RASTER2_SLOTS_FEW>(p, nblocks, s);
    else launch_raster2_slots<RASTER2_SLOTS>(p, nblocks, s);
}

void raster2_set_slots_override(int slots) { g_slots_override = slots > 0 ? slots : 0; }

}  // namespace scoup
