// raster.cu -- fused rasterise-and-aggregate kernel (the hot loop of Algorithm 1).
//
// One CTA of 256 threads per (view, 16x16 tile), one pixel per thread; warp w covers the 8x4
// pixel block at column 8*(w&1), row 4*(w>>1) of the tile (near-square blocks keep the number
// of (warp, Gaussian) pairs low for small footprints).  The tile reads the depth-ordered
// candidate list of the bin that contains it (bins are power-of-two squares of pixels,
// DESIGN.md §5) and walks it front to back:
//
//  refill   256 candidates at a time (their records fetched one round ahead with cp.async into
//           a per-thread staging slot) are tested against the tile (support box and the ellipse
//           band spans, conservatively, band_relevant) and stably compacted into a shared-memory
//           ring of records, so the ring stays in (depth, index) order;
//  batch    32 ring records at a time: each warp ballots the records that may touch its 8x4 block
//           (band_relevant) and, in order, every lane evaluates DESIGN.md §3 step PX on them -- square test, the
//           log2-domain quadratic form, the q <= 0 guard, alpha = min(0.99, o exp2_spec(q)), the
//           alpha >= 1/255 skip and the T(1-alpha) < 1e-4 stop -- giving the weights
//           e_i(v,p) = alpha_i T of PAPER.md Eq. 2, bit-identical to the CPU oracle.
//           Control flow is warp-uniform (one uniform branch per group of RGROUP records); the
//           per-lane decisions are predicates/selects.  The T-independent part (dx, dy, q,
//           o exp2_spec(q)) of records 2i and 2i+1 is evaluated together in paired FP32
//           (FADD2/FMUL2/FFMA2: two independent IEEE round-to-nearest ops per instruction, so
//           each half is bit-identical to the scalar spec); only the T chain runs per record.
//
// Aggregation (Eq. 5; Algorithm 1 lines 8-10), for all nlev semantic
// levels of the pass at once (the levels share every fragment, only
// the region maps differ): pixels are grouped by their tuple of region ids (one
// per level) into at most MAX_SLOTS tile slots; per warp and slot group the per-pixel weights of
// the batch are summed with a 31-shuffle transpose-reduction (lane l ends with the sum for the
// l-th batch record), the group sums of all warps are combined per (slot, Gaussian) in shared
// memory, and only then global reductions go out: nlev*S `red.global.add.f32` per
// (slot, Gaussian) into W_level[g][atom] (c * sum e) plus one per Gaussian into Z[g].  A tile
// with more than MAX_SLOTS distinct tuples falls back to per-pixel reductions.
#include "internal.cuh"

namespace scoup {

#ifdef RASTER_STATS
// measurement build only (-DRASTER_STATS): warp/sub-batch statistics of the production kernel
__device__ unsigned long long g_rstat[16];
#define RSTAT(i, v) atomicAdd(&g_rstat[i], (unsigned long long)(v))
#else
#define RSTAT(i, v) ((void)0)
#endif

namespace {

constexpr uint32_t KEY_NONE = 0xFFFFFFFFu;   // unassigned or outside the image
constexpr uint32_t SLOT_EMPTY = 0xFFFFFFFEu;  // slot-table sentinel
constexpr unsigned FULL = 0xffffffffu;
constexpr int QCAP = 512;                     // candidate ring (power of two >= 256 + 3 * SBATCH)
constexpr int NWARP = TILE_PIX / 32;
#ifndef RASTER_NSUB
#define RASTER_NSUB 2                         // sub-batches of BATCH records per barrier
#endif
constexpr int NSUB = RASTER_NSUB;
constexpr int SBATCH = NSUB * BATCH;          // records per super-batch (one barrier, one flush)
#ifndef RGROUP
#define RGROUP 8                              // records per warp-uniform branch in the pixel loop (even: pairs)
#endif

// Sum e[i] over the lanes in the group (all lanes if !MASKED); lane l returns the sum for i = l.
template <bool MASKED>
__device__ __forceinline__ float transpose_reduce(const float (&e)[BATCH], bool mine, int lane) {
    // (the adds of sums i and i+1 go pairwise through FADD2: the same two IEEE adds)
    float v[16];
    {
        const bool up = lane & 16;
#pragma unroll
        for (int i = 0; i < 16; i += 2) {
            float lo0 = e[i], hi0 = e[i + 16], lo1 = e[i + 1], hi1 = e[i + 17];
            if (MASKED) {
                lo0 = mine ? lo0 : 0.f; hi0 = mine ? hi0 : 0.f;
                lo1 = mine ? lo1 : 0.f; hi1 = mine ? hi1 : 0.f;
            }
            const float r0 = __shfl_xor_sync(FULL, up ? lo0 : hi0, 16);
            const float r1 = __shfl_xor_sync(FULL, up ? lo1 : hi1, 16);
            f2_split(f2_add(f2_pack(up ? hi0 : lo0, up ? hi1 : lo1), f2_pack(r0, r1)), v[i], v[i + 1]);
        }
    }
#pragma unroll
    for (int s = 8; s >= 2; s >>= 1) {
        const bool up = lane & s;
#pragma unroll
        for (int i = 0; i < s; i += 2) {
            const float r0 = __shfl_xor_sync(FULL, up ? v[i] : v[i + s], s);
            const float r1 = __shfl_xor_sync(FULL, up ? v[i + 1] : v[i + s + 1], s);
            f2_split(f2_add(f2_pack(up ? v[i + s] : v[i], up ? v[i + s + 1] : v[i + 1]), f2_pack(r0, r1)), v[i],
                     v[i + 1]);
        }
    }
    {
        const bool up = lane & 1;
        v[0] = (up ? v[1] : v[0]) + __shfl_xor_sync(FULL, up ? v[0] : v[1], 1);
    }
    return v[0];
}

// cp.async of 16 bytes (zero-filled when !pred) and group completion.
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool pred) {
    const uint32_t sa = (uint32_t)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(gmem), "r"(pred ? 16 : 0));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }

// Fallback aggregation of one fragment: every level's code of the pixel (row < 0: unassigned at
// that level, no W), and Z.  Scalars only, so the call needs no local-memory copies.
__device__ __noinline__ void overflow_reds(float* W, float* Z, const uint32_t* atoms, const float* coefs, int S,
                                           int L, int nlev, int64_t level_stride, uint32_t g, float ev, int64_t r0,
                                           int64_t r1, int64_t r2, int64_t r3) {
    atomicAdd(Z + g, ev);
    for (int l = 0; l < nlev; l++) {
        const int64_t row = l == 0 ? r0 : l == 1 ? r1 : l == 2 ? r2 : r3;
        if (row < 0) continue;
        float* Wl = W + (int64_t)l * level_stride;
        for (int s = 0; s < S; s++) {
            const uint32_t at = atoms ? __ldg(atoms + row + s) : (uint32_t)s;  // (no atoms: dense)
            if (at != NONE) atomicAdd(Wl + (int64_t)g * L + at, __fmul_rn(__ldg(coefs + row + s), ev));
        }
    }
}

static_assert(BATCH == 32, "batch = one record per lane (transpose-reduction, flush indexing)");
static_assert((SBATCH & (SBATCH - 1)) == 0 && SBATCH <= TILE_PIX, "super-batch: a power of two, <= one thread each");
static_assert(RGROUP % 2 == 0 && BATCH % RGROUP == 0, "records are evaluated in pairs");

struct Ring {
    // ring of candidate records; sub-batches start at multiples of BATCH, so each one is
    // contiguous in [0, QCAP)
    // (mx, my, r, o) and (qa, qb, qc, ycut) of records 2i and 2i+1, pair-interleaved so the
    // pixel loop evaluates two records per paired-FP32 instruction (FADD2 / FMUL2 / FFMA2):
    // p0[i] = (mx, mx', my, my'), p1[i] = (r, r', o, o'), p2[i] = (qa, qa', qb, qb'),
    // p3[i] = (qc, qc', ycut, ycut')
    float4 p0[QCAP / 2];
    float4 p1[QCAP / 2];
    float4 p2[QCAP / 2];
    float4 p3[QCAP / 2];
    float4 q2[QCAP];     // (support-box half-extents x, y, Gaussian id, sy)
    float4 q3[QCAP];     // band_relevant parameters
};

struct __align__(16) Smem {
    union {
        Ring r;
        uint32_t stage[TILE_PIX][MAX_LEV];  // setup only: tuples proposed by the warps' group leaders
    } u;
    // per (slot, record) sums of a batch, triple-buffered: batch i accumulates into buffer i % 3,
    // which is flushed after the batch's barrier; buffer (i+2) % 3 is zeroed meanwhile, so a
    // single barrier per batch separates every write from every read
    float acc[3][MAX_SLOTS * SBATCH];
    float accZ[3][SBATCH];
    // candidate records of the next refill round, fetched with cp.async one round ahead (slot t
    // is written and read by thread t only)
    float4 st0[TILE_PIX], st1[TILE_PIX], st2[TILE_PIX], st3[TILE_PIX];
    uint32_t slot_key[MAX_SLOTS][MAX_LEV];  // region id tuple of each slot
    uint32_t slot_atom[MAX_SLOTS][MAX_S];   // per slot: nlev codes of S slots each
    float slot_coef[MAX_SLOTS][MAX_S];
    int nstage;
    int wcnt[NWARP];
    int nslot;
    int overflow;
    unsigned long long contrib;
    unsigned long long tests;
    unsigned long long evals;
    unsigned long long reds;
};


#ifndef RASTER_MIN_BLOCKS
#define RASTER_MIN_BLOCKS 3
#endif
// NLEV1: a single semantic level (the BASELINE configs' default), so that every level loop and
// the tuple bookkeeping fold away; else 1..MAX_LEV levels from p.nlev.
// COUNT: the instrumented variant that also counts contributions and support tests (stats,
// contributions_out); the production variant skips both counters in the pixel loop.
template <bool COUNT, bool NLEV1>
__global__ void __launch_bounds__(TILE_PIX, RASTER_MIN_BLOCKS) raster_aggregate_kernel(const RasterParams p) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Smem& sm = *reinterpret_cast<Smem*>(smem_raw);
    const int ntiles = p.bn.tiles_x * p.bn.tiles_y;
    const int view = blockIdx.x / ntiles, tile = blockIdx.x - view * ntiles;
    const int tx = tile % p.bn.tiles_x, ty = tile / p.bn.tiles_x;
    const int64_t gtile = (int64_t)view * ntiles + tile;
    if (p.chunk > 0 && !p.tile_live[gtile]) return;  // every pixel finished in an earlier chunk
    const int bin = ((ty * TILE) >> p.bn.bshy) * p.bn.bins_x + ((tx * TILE) >> p.bn.bshx);
    const uint2 range = p.ranges[view * p.bn.nbins() + bin];
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const int wx0 = tx * TILE + 8 * (warp & 1), wy0 = ty * TILE + 4 * (warp >> 1);
    const int x = wx0 + (lane & 7), y = wy0 + (lane >> 3);
    const int Wd = p.width, Hd = p.height;
    const bool inside = x < Wd && y < Hd;
    float* Tpix = p.Tstate + (int64_t)view * Wd * Hd + (int64_t)y * Wd + x;
    if (range.x >= range.y) {  // nothing of this chunk reaches the tile
        if (p.chunk == 0) {
            if (inside) *Tpix = 1.0f;
            if (t == 0) p.tile_live[gtile] = 1;
        }
        return;
    }
#ifdef RASTER_STATS
    if (threadIdx.x == 0) { RSTAT(13, 1); RSTAT(14, range.y - range.x); }
#endif
    // software-pipelined candidate fetch: the records of round k+1 are in flight (cp.async)
    // while round k's batches are evaluated; the list indices are loaded one round further ahead.
    // The first round is issued before the slot setup, whose region-id and code loads then
    // overlap its two dependent global latencies (list index, then record).
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
    uint32_t e_next = cursor + TILE_PIX + t < range.y ? __ldg(p.eval + cursor + TILE_PIX + t) : 0u;
    const int nlev = NLEV1 ? 1 : p.nlev;
    float* const pf0 = reinterpret_cast<float*>(sm.u.r.p0);
    float* const pf1 = reinterpret_cast<float*>(sm.u.r.p1);
    float* const pf2 = reinterpret_cast<float*>(sm.u.r.p2);
    float* const pf3 = reinterpret_cast<float*>(sm.u.r.p3);
    // record at ring position pos: element (pos >> 1) * 4 + (pos & 1) (+ 2 for the second pair)
    auto put_pair_rec = [&](uint32_t pos, const float4& r0, const float4& r1) {
        const uint32_t b = (pos >> 1) * 4 + (pos & 1);
        pf0[b] = r0.x; pf0[b + 2] = r0.y; pf1[b] = r0.z; pf1[b + 2] = r0.w;
        pf2[b] = r1.x; pf2[b + 2] = r1.y; pf3[b] = r1.z; pf3[b + 2] = r1.w;
    };
    auto get_rec0 = [&](uint32_t pos) {
        const uint32_t b = (pos >> 1) * 4 + (pos & 1);
        return make_float4(pf0[b], pf0[b + 2], pf1[b], pf1[b + 2]);
    };
    float4* const q2 = sm.u.r.q2;
    float4* const q3 = sm.u.r.q3;
    // pixel-centre rectangles of the tile and of this warp's 8x4 block (clipped to the image)
    const float TX0 = (float)(tx * TILE) + 0.5f, TY0 = (float)(ty * TILE) + 0.5f;
    const float TX1 = (float)(min(tx * TILE + TILE, Wd) - 1) + 0.5f;
    const float TY1 = (float)(min(ty * TILE + TILE, Hd) - 1) + 0.5f;
    const float WX0 = (float)wx0 + 0.5f, WY0 = (float)wy0 + 0.5f;
    const float WX1 = (float)(min(wx0 + 8, Wd) - 1) + 0.5f, WY1 = (float)(min(wy0 + 4, Hd) - 1) + 0.5f;

    // ---- setup: region id tuple of my pixel, tile slot table (distinct tuples), slot codes
    uint32_t key[MAX_LEV];
#pragma unroll
    for (int l = 0; l < MAX_LEV; l++) {
        key[l] = KEY_NONE;
        if (l < nlev && inside) {
            uint32_t rid = __ldg(p.region_ids[view][l] + (int64_t)y * Wd + x);
            if (rid != NONE && rid >= (uint32_t)p.num_regions[view][l]) {
                latch_error(p.err, ERR_REGION,
                            ((long long)l << 48) + p.pixel_base[view] + (int64_t)y * Wd + x);
                rid = NONE;
            }
            key[l] = rid;
        }
    }
    if (t == 0) { sm.nslot = 0; sm.nstage = 0; sm.overflow = 0; sm.contrib = 0ull; sm.tests = 0ull; sm.evals = 0ull; sm.reds = 0ull; }
    if (t < MAX_SLOTS) sm.slot_key[t][0] = SLOT_EMPTY;
    for (int i = t; i < 3 * MAX_SLOTS * SBATCH; i += TILE_PIX) (&sm.acc[0][0])[i] = 0.f;
    for (int i = t; i < 3 * SBATCH; i += TILE_PIX) (&sm.accZ[0][0])[i] = 0.f;
    unsigned grp = FULL;
#pragma unroll
    for (int l = 0; l < MAX_LEV; l++)
        if (l < nlev) grp &= __match_any_sync(FULL, key[l]);  // lanes with my whole tuple
    __syncthreads();
    int slot = 0;
    if (NLEV1) {
        // one region id per pixel: the warp's group leader claims (or finds) its slot by CAS
        const int leader = __ffs(grp) - 1;
        int sl = -1;
        if (lane == leader) {
            for (int q = 0; q < MAX_SLOTS; q++) {
                const uint32_t old = atomicCAS(&sm.slot_key[q][0], SLOT_EMPTY, key[0]);
                if (old == SLOT_EMPTY || old == key[0]) { sl = q; break; }
            }
            if (sl < 0) sm.overflow = 1;
            else atomicMax(&sm.nslot, sl + 1);
        }
        slot = max(0, __shfl_sync(FULL, sl, leader));
        __syncthreads();
    } else {
        if (lane == __ffs(grp) - 1) {  // one proposal per distinct tuple per warp
            const int k = atomicAdd(&sm.nstage, 1);
            for (int l = 0; l < MAX_LEV; l++) sm.u.stage[k][l] = key[l];
        }
        __syncthreads();
        if (t == 0) {  // deduplicate the (few) proposals into the slot table
            int ns = 0;
            const int np = sm.nstage;
            for (int k = 0; k < np; k++) {
                int f = -1;
                for (int q = 0; q < ns && f < 0; q++) {
                    bool eq = true;
                    for (int l = 0; l < nlev; l++) eq = eq && sm.slot_key[q][l] == sm.u.stage[k][l];
                    if (eq) f = q;
                }
                if (f < 0) {
                    if (ns == MAX_SLOTS) { sm.overflow = 1; break; }
                    for (int l = 0; l < MAX_LEV; l++) sm.slot_key[ns][l] = sm.u.stage[k][l];
                    ns++;
                }
            }
            sm.nslot = ns;
        }
        __syncthreads();
        if (!sm.overflow) {
            for (int q = 0; q < sm.nslot; q++) {
                bool eq = true;
                for (int l = 0; l < nlev; l++) eq = eq && sm.slot_key[q][l] == key[l];
                if (eq) { slot = q; break; }
            }
        }
    }
    const int nslot = sm.nslot;
    const bool overflow = sm.overflow != 0;
    const int S = p.S;
    const int LS = nlev * S;  // W updates per (slot, Gaussian): every level's code
    const int ls_log2 = (LS & (LS - 1)) == 0 ? __ffs(LS) - 1 : -1;
    const int s_log2 = (S & (S - 1)) == 0 ? __ffs(S) - 1 : -1;
    // ceil(2^32 / d) for the flush's divisions by d = LS, S when they are not powers of two:
    // __umulhi(i, m) == i / d exactly when i * d < 2^32
    const uint32_t ls_magic = 0xFFFFFFFFu / (uint32_t)LS + 1u, s_magic = 0xFFFFFFFFu / (uint32_t)S + 1u;
    for (int i = t; i < (p.dense ? 0 : nslot * LS); i += TILE_PIX) {  // (dense: read in the flush)
        const int q = i / LS, ls = i - q * LS, l = ls / S, s = ls - l * S;
        const uint32_t k = sm.slot_key[q][l];
        uint32_t a = NONE;
        float c = 0.f;
        if (k != KEY_NONE) {
            const int64_t row = (p.code_row0[view][l] + (int64_t)k) * S + s;
            a = __ldg(p.code_atoms + row);
            c = __ldg(p.code_coefs + row);
        }
        sm.slot_atom[q][ls] = a;
        sm.slot_coef[q][ls] = c;
    }
    // (slot codes are first read after a later barrier; the ring overwrites the staging area
    // only after the barrier of the first refill round)

    const float px = __fadd_rn((float)x, 0.5f), py = __fadd_rn((float)y, 0.5f);
    // transmittance; T < 1e-4 marks a finished pixel (T = 0 outside the image; at the stop of
    // DESIGN.md §4 R9, T(1 - alpha) < 1e-4, T keeps that product) -- a live pixel's T never drops
    // below 1e-4, and a finished one can only shrink, so it never passes the stop test again
    float T = !inside ? 0.0f : (p.chunk == 0 ? 1.0f : *Tpix);
    uint32_t cnt = 0, tests = 0, wevals = 0, nred = 0;
    const int L = p.L;
    const unsigned lanemask_lt = (1u << lane) - 1u;

    uint32_t q_head = 0, q_count = 0;
    int buf = 0;
    while (true) {
        // ---- refill the ring: candidates with their warp masks (stable compaction)
        while (q_count < (uint32_t)SBATCH && cursor < range.y) {
            const uint32_t idx = cursor + t;
            cp_async_wait_all();  // this round's records (my staging slot)
            const float4 r0 = sm.st0[t], r1 = sm.st1[t], r2 = sm.st2[t], r3 = sm.st3[t];
            const bool acc = idx < range.y && band_relevant(r0, r2, r3, TX0, TX1, TY0, TY1);
            {   // start the next round's fetch (my slot is free again)
                const uint32_t nidx = cursor + TILE_PIX + t;
                prefetch(e_next, nidx < range.y);
                e_next = nidx + TILE_PIX < range.y ? __ldg(p.eval + nidx + TILE_PIX) : 0u;
            }
            const unsigned bal = __ballot_sync(FULL, acc);
            if (lane == 0) sm.wcnt[warp] = __popc(bal);
            __syncthreads();
            uint32_t off = 0, tot = 0;
#pragma unroll
            for (int w = 0; w < NWARP; w++) {
                const uint32_t c = (uint32_t)sm.wcnt[w];
                off += (w < warp) ? c : 0u;
                tot += c;
            }
            if (acc) {
                const uint32_t pos = (q_head + q_count + off + __popc(bal & lanemask_lt)) & (QCAP - 1);
                put_pair_rec(pos, r0, r1);
                q2[pos] = r2;
                q3[pos] = r3;
            }
            q_count += tot;
            cursor += TILE_PIX;
#ifdef RASTER_STATS
            if (t == 0) { RSTAT(9, 1); RSTAT(10, tot); }
#endif
            __syncthreads();
        }
        if (q_count == 0) break;
        // a super-batch: up to NSUB sub-batches of BATCH records (each starts at a multiple of
        // BATCH in the ring, so it is contiguous), evaluated back to back by every warp, then ONE
        // barrier and one flush for all of them
        const uint32_t n = min((uint32_t)SBATCH, q_count);
        const int nsub = (int)((n + BATCH - 1) / BATCH);
#ifdef RASTER_STATS
        if (t == 0) { RSTAT(11, 1); RSTAT(12, n); }
#endif
        if (n % BATCH) {
            // the tile's last, partial sub-batch: the ring slots past it hold stale records, which
            // the pixel loop (it evaluates whole record groups without a per-record mask test)
            // must see as empty -- a negative support radius fails every square test
            if ((uint32_t)t >= n && t < nsub * BATCH) {
                const uint32_t pos = (q_head + (uint32_t)t) & (QCAP - 1);
                pf1[(pos >> 1) * 4 + (pos & 1)] = -1.0f;
            }
            __syncthreads();
        }
        bool any_sb = false;
#pragma unroll 1
        for (int sb = 0; sb < nsub; sb++) {
        const uint32_t sh = (q_head + (uint32_t)(sb * BATCH)) & (QCAP - 1);  // sub-batch head
        const uint32_t nsb = min((uint32_t)BATCH, n - (uint32_t)(sb * BATCH));
        // ---- per-warp mask of sub-batch records that may touch this warp's 8x4 block
        const bool warp_done = __all_sync(FULL, !(T >= K_TMIN));
        bool rel = false;
        if (!warp_done && (uint32_t)lane < nsb)
            rel = band_relevant(get_rec0(sh + lane), q2[sh + lane], q3[sh + lane], WX0, WX1, WY0, WY1);
        const unsigned mask = __ballot_sync(FULL, rel);
#ifdef RASTER_STATS
        if (lane == 0 && !warp_done) {
            int ng = 0;
            for (int g0 = 0; g0 < BATCH; g0 += RGROUP) ng += ((mask >> g0) & ((1u << RGROUP) - 1u)) ? 1 : 0;
            RSTAT(0, 1);
            RSTAT(1 + ng, 1);          // [1..5]: 0..4 active groups
            RSTAT(6, grp == FULL);
            RSTAT(7, __popc(mask));
            RSTAT(8, nsb);
        }
#endif

        // ---- rasterise: e[j] for sub-batch record j, in depth order (DESIGN.md §3 PX).
        // Records go in groups of RGROUP with one warp-uniform branch per group: inside a group
        // there is no control flow, so the T-independent work of the next record (loads, q,
        // exp2_spec) overlaps the T update of the current one.  A record outside the warp's
        // mask is a no-op (its `sq` is false).
        float e[BATCH];
        uint32_t cbits = 0u, tbits = 0u;  // per record: contributed / tested (support square)
        const ulonglong2* b0 = reinterpret_cast<const ulonglong2*>(sm.u.r.p0) + (sh >> 1);
        const ulonglong2* b1 = reinterpret_cast<const ulonglong2*>(sm.u.r.p1) + (sh >> 1);
        const ulonglong2* b2 = reinterpret_cast<const ulonglong2*>(sm.u.r.p2) + (sh >> 1);
        const ulonglong2* b3 = reinterpret_cast<const ulonglong2*>(sm.u.r.p3) + (sh >> 1);
#pragma unroll
        for (int j = 0; j < BATCH; j++) e[j] = 0.f;
#pragma unroll
        for (int g0 = 0; g0 < BATCH; g0 += RGROUP)
        if ((mask >> g0) & ((1u << RGROUP) - 1u)) {
#pragma unroll
        for (int j = g0; j < g0 + RGROUP; j += 2) {
            // T-independent part of records j and j+1 in paired FP32 (each half is the exact
            // DESIGN.md §3 scalar operation, round-to-nearest, no contraction)
            const ulonglong2 A0 = b0[j >> 1], A1 = b1[j >> 1], A2 = b2[j >> 1], A3 = b3[j >> 1];
            const f2 dx = f2_rsub(A0.x, px), dy = f2_rsub(A0.y, py);      // px - mx, py - my
            const f2 q = f2_fma(dx, f2_fma(A2.x, dx, f2_mul(A2.y, dy)), f2_mul(f2_mul(A3.x, dy), dy));
            const f2 ex = exp2_spec2(q);
            float mx_lo, mx_hi;
            f2_split(f2_mul(A1.y, ex), mx_lo, mx_hi);                       // o * exp2_spec(q)
            const float al0 = fminf(K_ACLAMP, mx_lo), al1 = fminf(K_ACLAMP, mx_hi);
            float om0, om1;
            f2_split(f2_rsub(f2_pack(al0, al1), 1.0f), om0, om1);            // 1 - alpha
            float dx0, dx1, dy0, dy1, q0, q1, r0, r1, y0, y1;
            f2_split(dx, dx0, dx1);
            f2_split(dy, dy0, dy1);
            f2_split(q, q0, q1);
            f2_split(A1.x, r0, r1);
            f2_split(A3.y, y0, y1);
#pragma unroll
            for (int h = 0; h < 2; h++) {
                const float dxh = h ? dx1 : dx0, dyh = h ? dy1 : dy0, qh = h ? q1 : q0, rh = h ? r1 : r0;
                const float yh = h ? y1 : y0, al = h ? al1 : al0, om = h ? om1 : om0;
                const int jj = j + h;
                // (a finished pixel, T < 1e-4, needs no test of its own: its Tn <= T < 1e-4 makes
                // every later fragment a non-contributing stop that leaves T < 1e-4)
                // (the record's warp-mask bit is only needed for the support-test count: a
                // record outside the mask cannot pass the alpha test anywhere in the block --
                // band_relevant is conservative -- so it is a no-op for every lane)
                const bool sq = (!COUNT || ((mask >> jj) & 1u)) && fabsf(dxh) <= rh && fabsf(dyh) <= rh;
                const bool active = COUNT && T >= K_TMIN;
                const float Tn = __fmul_rn(T, om);
                const bool pass = sq && !(qh > 0.f) && qh >= yh && al >= K_AMIN;
                const bool con = pass && !(Tn < K_TMIN);
                e[jj] = con ? __fmul_rn(al, T) : 0.f;
                T = pass ? Tn : T;  // pass && !con: the pixel ends here (Tn < 1e-4); a short chain
                if (COUNT && con) cbits |= 1u << jj;
                if (COUNT && sq && active) tbits |= 1u << jj;
            }
        }
        }
        // (uncounted: the reductions run whenever the warp evaluated a record; all-zero sums add
        // nothing)
        const bool any = COUNT ? cbits != 0u : mask != 0u;
        any_sb = any_sb || any;
        cnt += __popc(cbits);
        tests += __popc(tbits);
        if (COUNT) {  // records this warp evaluated (whole groups: the branch is per group)
            unsigned gm = 0u;
#pragma unroll
            for (int g0 = 0; g0 < BATCH; g0 += RGROUP) gm += ((mask >> g0) & ((1u << RGROUP) - 1u)) ? RGROUP : 0u;
            wevals += gm;
        }
        if (overflow && any) {
            // per-pixel reductions straight from the code table (tiles with > MAX_SLOTS tuples)
#pragma unroll
            for (int j = 0; j < BATCH; j++) {
                if (e[j] > 0.f) {
                    int64_t rw[MAX_LEV];  // my code rows (region ids re-read: a rare path)
#pragma unroll
                    for (int l = 0; l < MAX_LEV; l++) {
                        uint32_t k = KEY_NONE;
                        if (l < nlev) k = __ldg(p.region_ids[view][l] + (int64_t)y * Wd + x);
                        rw[l] = (k != NONE && k < (uint32_t)p.num_regions[view][l])
                                    ? (p.code_row0[view][l] + (int64_t)k) * S : -1;
                    }
                    overflow_reds(p.W, p.Z, p.dense ? nullptr : p.code_atoms, p.code_coefs, S, L, nlev, p.W_level_stride,
                                  __float_as_uint(q2[sh + j].z), e[j], rw[0], rw[1], rw[2], rw[3]);
                }
            }
        }

        if (!overflow) {
            // ---- per (warp, slot group) transpose-reduction, then shared accumulation
            if (__any_sync(FULL, any)) {
                // lane l ends with the group's sum for sub-batch record l
                const bool mine_rel = (mask >> lane) & 1u;
                const int col = sb * BATCH + lane;  // record column in the super-batch sums
                if (grp == FULL) {
                    const float v = transpose_reduce<false>(e, true, lane);
                    if (mine_rel && v != 0.f) {
                        atomicAdd(&sm.acc[buf][slot * SBATCH + col], v);
                        atomicAdd(&sm.accZ[buf][col], v);
                    }
                } else {
                    float zsum = 0.f;
                    unsigned todo = FULL;
                    while (todo) {
                        const int l = __ffs(todo) - 1;
                        const unsigned g2 = __shfl_sync(FULL, grp, l);
                        const int q = __shfl_sync(FULL, slot, l);
                        todo &= ~g2;
                        const float v = transpose_reduce<true>(e, (g2 >> lane) & 1u, lane);
                        if (mine_rel && v != 0.f) atomicAdd(&sm.acc[buf][q * SBATCH + col], v);
                        zsum += mine_rel ? v : 0.f;
                    }
                    if (zsum != 0.f) atomicAdd(&sm.accZ[buf][col], zsum);
                }
            }
        }
        }  // sub-batches
        (void)any_sb;
        // B: the super-batch's sums are complete; also the termination vote (all pixels finished)
        const int alive = __syncthreads_count(T >= K_TMIN);
        if (!overflow) {
            // ---- flush: nlev*S reds per (slot, Gaussian) into W_level, one per Gaussian into Z
            // one red of W update ls (level l = ls / S, code slot ls % S) of (slot q, record j)
            auto gid_of = [&](int j) { return __float_as_uint(q2[(q_head + (uint32_t)j) & (QCAP - 1)].z); };
            auto red_one = [&](int q, int j, int ls, float v) {
                const int l = s_log2 >= 0 ? ls >> s_log2 : (int)__umulhi((uint32_t)ls, s_magic);
                uint32_t a;
                float c;
                if (p.dense) {  // dense features (Eq. 3 baseline): slot s is atom s, from the table
                    a = (uint32_t)(ls - l * S);
                    const uint32_t k = sm.slot_key[q][l];
                    c = k != KEY_NONE && v > 0.f ? __ldg(p.code_coefs + (p.code_row0[view][l] + (int64_t)k) * S + a)
                                                 : 0.f;
                    if (k == KEY_NONE) a = NONE;
                } else {
                    a = sm.slot_atom[q][ls];
                    c = sm.slot_coef[q][ls];
                }
                if (COUNT && v > 0.f && a != NONE) nred++;
                if (v > 0.f && a != NONE)
                    atomicAdd(p.W + (int64_t)l * p.W_level_stride + (int64_t)gid_of(j) * L + a, __fmul_rn(c, v));
            };
            const int ncol = nsub * BATCH;  // record columns in use (the rest of each slot row is zero)
            if (ls_log2 >= 0) {
                // nlev * S a power of two (every single-level BASELINE config): the CTA's threads
                // sweep all (slot, record, update) items, LS consecutive threads per sum
                const int nitems = nslot * SBATCH * LS;
                for (int i = t; i < nitems; i += TILE_PIX) {
                    const int u = i >> ls_log2, j = u & (SBATCH - 1);
                    if (j < ncol) red_one(u / SBATCH, j, i & (LS - 1), sm.acc[buf][u]);
                }
            } else {
                // (u = i / LS by multiply-high, exact for i * LS < 2^32: every flush index while
                // LS <= 2048; SBATCH is a power of two.  A per-warp ballot over the (slot, record)
                // sums that skips the zero ones was measured slower: indoor 106 -> 128 ms)
                const int nitems = nslot * SBATCH * LS;
                for (int i = t; i < nitems; i += TILE_PIX) {
                    const uint32_t u = LS <= 2048 ? __umulhi((uint32_t)i, ls_magic) : (uint32_t)i / (uint32_t)LS;
                    const int j = (int)(u & (SBATCH - 1));
                    if (j < ncol) red_one((int)(u / SBATCH), j, i - (int)u * LS, sm.acc[buf][u]);
                }
            }
            if (t < ncol) {
                const float z = sm.accZ[buf][t];
                if (COUNT && z > 0.f) nred++;
                if (z > 0.f) atomicAdd(p.Z + gid_of(t), z);
            }
            // zero the buffer of super-batch i+2 (flushed in super-batch i-1, before this barrier)
            const int bz = buf == 0 ? 2 : buf - 1;
            for (int i = t; i < nslot * SBATCH; i += TILE_PIX) sm.acc[bz][i] = 0.f;
            if (t < SBATCH) sm.accZ[bz][t] = 0.f;
        }
        // (no second barrier: the next refill writes only ring slots past this super-batch, and
        // the next super-batch accumulates into another buffer)
        q_head = (q_head + n) & (QCAP - 1);
        q_count -= n;
        buf = buf == 2 ? 0 : buf + 1;
        if (alive == 0) break;
    }

    cp_async_wait_all();  // no copy may land in shared memory after the CTA retires

    // carry the per-pixel state to the next chunk
    if (inside) *Tpix = T;
    const int live = __syncthreads_count(T >= K_TMIN);
    if (t == 0) p.tile_live[gtile] = live > 0 ? 1 : 0;

    // contributions (terms of Eq. 5's sum) and support tests
    const unsigned c = COUNT ? __reduce_add_sync(FULL, cnt) : 0u;
    if (lane == 0 && c) atomicAdd(&sm.contrib, (unsigned long long)c);
    if (COUNT) {
        const unsigned ts = __reduce_add_sync(FULL, tests);
        if (lane == 0 && ts) atomicAdd(&sm.tests, (unsigned long long)ts);
        if (lane == 0 && wevals) atomicAdd(&sm.evals, 32ull * wevals);
        const unsigned rs = __reduce_add_sync(FULL, nred);
        if (lane == 0 && rs) atomicAdd(&sm.reds, (unsigned long long)rs);
    }
    __syncthreads();
    if (t == 0) {
        if (sm.contrib) {
            atomicAdd(p.contrib_ctr, sm.contrib);
            if (p.contrib_out[view]) atomicAdd(reinterpret_cast<unsigned long long*>(p.contrib_out[view]), sm.contrib);
        }
        if (COUNT && sm.tests) atomicAdd(p.support_ctr, sm.tests);
        if (COUNT && sm.evals) atomicAdd(p.lane_eval_ctr, sm.evals);
        if (COUNT && sm.reds) atomicAdd(p.red_ctr, sm.reds);
    }
}

}  // namespace

#ifdef RASTER_STATS
extern "C" int scoup_debug_raster_stats(unsigned long long* out, int reset) {
    cudaDeviceSynchronize();
    cudaMemcpyFromSymbol(out, g_rstat, sizeof(unsigned long long) * 16);
    if (reset) {
        unsigned long long z[16] = {};
        cudaMemcpyToSymbol(g_rstat, z, sizeof(z));
    }
    return 0;
}
#endif

void launch_raster(const RasterParams& p, cudaStream_t s) {
    const int ntiles = p.bn.tiles_x * p.bn.tiles_y * p.nviews;
    if (ntiles <= 0) return;
    static_assert(3 * (sizeof(Smem) + 1024) <= 228 * 1024, "three CTAs per SM must fit the 228 KB shared memory");
    static bool attr_set = false;  // the opt-in above 48 KB of dynamic shared memory, once
    if (!attr_set) {
        cudaFuncSetAttribute(raster_aggregate_kernel<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)sizeof(Smem));
        cudaFuncSetAttribute(raster_aggregate_kernel<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)sizeof(Smem));
        cudaFuncSetAttribute(raster_aggregate_kernel<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)sizeof(Smem));
        cudaFuncSetAttribute(raster_aggregate_kernel<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)sizeof(Smem));
        attr_set = true;
    }
    const size_t smem = sizeof(Smem);
    if (p.nlev == 1) {
        if (p.count_tests)
            raster_aggregate_kernel<true, true><<<ntiles, TILE_PIX, smem, s>>>(p);
        else
            raster_aggregate_kernel<false, true><<<ntiles, TILE_PIX, smem, s>>>(p);
    } else {
        if (p.count_tests)
            raster_aggregate_kernel<true, false><<<ntiles, TILE_PIX, smem, s>>>(p);
        else
            raster_aggregate_kernel<false, false><<<ntiles, TILE_PIX, smem, s>>>(p);
    }
}

}  // namespace scoup
