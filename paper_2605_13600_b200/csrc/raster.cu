// raster.cu -- fused rasterise-and-aggregate kernel (the hot loop of Algorithm 1).
//
// One CTA of 256 threads per 16x16 tile, one pixel per thread (natural row-major order, so
// a warp is a 16x2 pixel block).  The tile's Gaussian list (depth order) is walked in
// batches of 32 records staged in shared memory (double-buffered, prefetched by warp 0).
// Per pixel and Gaussian the thread applies DESIGN.md §3 step PX -- square support, the
// log2-domain quadratic form, the y <= 0 guard, alpha = min(0.99, o exp2_spec(y)), the
// alpha >= 1/255 skip and the T(1-alpha) < 1e-4 stop -- giving e_i(v,p) = alpha_i T
// (Eq. 2) bit-identical to the CPU oracle.
//
// Aggregation (Eq. 5; Algorithm 1 lines 8-10): the 32 per-pixel
// weights of a batch are summed over the pixels of each (warp, region) group with a
// 31-shuffle transpose-reduction (lane l ends with the group's sum for Gaussian l), the
// group sums of all warps are combined per (tile region, Gaussian) in shared memory, and
// only then do global reductions go out: S `red.global.add.f32` per (tile region,
// Gaussian) into W[g][atom] (value c * sum e) plus one per Gaussian into Z[g].  A tile with
// more than MAX_SLOTS distinct regions falls back to per-pixel reductions.
#include "internal.cuh"

namespace scoup {

namespace {

constexpr uint32_t KEY_NONE = 0xFFFFFFFFu;   // unassigned or outside the image
constexpr uint32_t SLOT_EMPTY = 0xFFFFFFFEu;  // hash-table sentinel (never a region id here)
constexpr unsigned FULL = 0xffffffffu;

// DESIGN.md §3 exp2_spec for ycut <= y <= 0 (the caller's conservative prune guarantees
// y >= ycut > -64, so the oracle's y < -64 branch is unreachable here).
__device__ __forceinline__ float exp2_spec(float y) {
    const float magic = 0x1.8p23f;
    float t = __fadd_rn(y, magic);  // round-half-even to an integer
    float kf = __fsub_rn(t, magic);
    float f = __fsub_rn(y, kf);
    float p = 0x1.4258dap-13f;
    p = __fmaf_rn(p, f, 0x1.5f44dep-10f);
    p = __fmaf_rn(p, f, 0x1.3b2cc4p-7f);
    p = __fmaf_rn(p, f, 0x1.c6aed6p-5f);
    p = __fmaf_rn(p, f, 0x1.ebfbdcp-3f);
    p = __fmaf_rn(p, f, 0x1.62e430p-1f);
    p = __fmaf_rn(p, f, 1.0f);
    // ldexp(p, k): bits(t) << 23 == k << 23 (mod 2^32) for t = 1.5*2^23 + k
    return __int_as_float(__float_as_int(p) + (__float_as_int(t) << 23));
}

// Sum e[j] over the lanes of `grp` (all lanes if grp == FULL); lane l returns the sum for j = l.
template <bool MASKED>
__device__ __forceinline__ float transpose_reduce(const float (&e)[BATCH], bool mine, int lane) {
    float v[16];
    {
        const bool up = lane & 16;
#pragma unroll
        for (int i = 0; i < 16; i++) {
            float lo = e[i], hi = e[i + 16];
            if (MASKED) { lo = mine ? lo : 0.f; hi = mine ? hi : 0.f; }
            float send = up ? lo : hi;
            float keep = up ? hi : lo;
            v[i] = keep + __shfl_xor_sync(FULL, send, 16);
        }
    }
#pragma unroll
    for (int s = 8; s >= 1; s >>= 1) {
        const bool up = lane & s;
#pragma unroll
        for (int i = 0; i < s; i++) {
            float send = up ? v[i] : v[i + s];
            float keep = up ? v[i + s] : v[i];
            v[i] = keep + __shfl_xor_sync(FULL, send, s);
        }
    }
    return v[0];
}

struct __align__(16) Smem {
    float4 rec0[2][BATCH];
    float4 rec1[2][BATCH];
    uint32_t gid[2][BATCH];
    float acc[2][MAX_SLOTS * BATCH];
    float accZ[2][BATCH];
    uint32_t slot_key[MAX_SLOTS];
    uint32_t slot_atom[MAX_SLOTS][MAX_S];
    float slot_coef[MAX_SLOTS][MAX_S];
    int nslot;
    int overflow;
    unsigned long long contrib;
    unsigned long long tests;
};

__device__ __forceinline__ void smem_add(float* p, float v) { atomicAdd(p, v); }

__global__ void __launch_bounds__(TILE_PIX, 3) raster_aggregate_kernel(const RasterParams p) {
    __shared__ Smem sm;
    const int tile = blockIdx.x;
    const uint2 range = p.ranges[tile];
    if (range.x >= range.y) return;
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const int tx = tile % p.tiles_x, ty = tile / p.tiles_x;
    const int x = tx * TILE + (t & (TILE - 1)), y = ty * TILE + (t >> 4);
    const int Wd = p.cam.width, Hd = p.cam.height;
    const bool inside = x < Wd && y < Hd;

    // ---- setup: region key of my pixel, tile slot table, slot codes
    uint32_t key = KEY_NONE;
    if (inside) {
        uint32_t rid = __ldg(p.region_ids + (int64_t)y * Wd + x);
        if (rid != NONE && rid >= (uint32_t)p.num_regions) {
            latch_error(p.err, ERR_REGION, p.pixel_base + (int64_t)y * Wd + x);
            rid = NONE;
        }
        key = rid;
    }
    if (t < MAX_SLOTS) sm.slot_key[t] = SLOT_EMPTY;
    if (t == 0) { sm.nslot = 0; sm.overflow = 0; sm.contrib = 0ull; sm.tests = 0ull; }
    for (int i = t; i < 2 * MAX_SLOTS * BATCH; i += TILE_PIX) (&sm.acc[0][0])[i] = 0.f;
    if (t < 2 * BATCH) (&sm.accZ[0][0])[t] = 0.f;
    // first batch of records (warp 0)
    const uint32_t nent = range.y - range.x;
    if (warp == 0) {
        uint32_t g = 0;
        float4 r0 = make_float4(0.f, 0.f, -1.f, 0.f), r1 = make_float4(0.f, 0.f, 0.f, 0.f);
        if ((uint32_t)lane < nent) {
            g = __ldg(p.eval + range.x + lane);
            r0 = __ldg(p.rec0 + g);
            r1 = __ldg(p.rec1 + g);
        }
        sm.gid[0][lane] = g;
        sm.rec0[0][lane] = r0;
        sm.rec1[0][lane] = r1;
    }
    __syncthreads();
    const unsigned grp = __match_any_sync(FULL, key);
    const int leader = __ffs(grp) - 1;
    int slot = -1;
    if (lane == leader) {
        for (int q = 0; q < MAX_SLOTS; q++) {
            uint32_t old = atomicCAS(&sm.slot_key[q], SLOT_EMPTY, key);
            if (old == SLOT_EMPTY || old == key) { slot = q; break; }
        }
        if (slot < 0) sm.overflow = 1;
        else atomicMax(&sm.nslot, slot + 1);
    }
    slot = __shfl_sync(FULL, slot, leader);
    __syncthreads();
    const int nslot = sm.nslot;
    const bool overflow = sm.overflow != 0;
    const int S = p.S;
    for (int i = t; i < nslot * S; i += TILE_PIX) {
        const int q = i / S, s = i - q * S;
        const uint32_t k = sm.slot_key[q];
        uint32_t a = NONE;
        float c = 0.f;
        if (k != KEY_NONE) {
            const int64_t row = (p.code_row0 + (int64_t)k) * S + s;
            a = __ldg(p.code_atoms + row);
            c = __ldg(p.code_coefs + row);
        }
        sm.slot_atom[q][s] = a;
        sm.slot_coef[q][s] = c;
    }
    // no barrier needed yet: slot codes are first read after the first B1 barrier

    const float px = __fadd_rn((float)x, 0.5f), py = __fadd_rn((float)y, 0.5f);
    float T = 1.0f;
    bool done = !inside;
    uint32_t cnt = 0, tests = 0;
    float* Wm = p.W;
    const int L = p.L;

    int buf = 0;
    for (uint32_t base = range.x; base < range.y; base += BATCH, buf ^= 1) {
        const uint32_t n = min((uint32_t)BATCH, range.y - base);
        // prefetch next batch's records into registers (warp 0)
        uint32_t ng = 0;
        float4 nr0 = make_float4(0.f, 0.f, -1.f, 0.f), nr1 = make_float4(0.f, 0.f, 0.f, 0.f);
        const uint32_t nbase = base + BATCH;
        if (warp == 0 && nbase + lane < range.y) {
            ng = __ldg(p.eval + nbase + lane);
            nr0 = __ldg(p.rec0 + ng);
            nr1 = __ldg(p.rec1 + ng);
        }

        // ---- rasterise: e[j] for the batch (DESIGN.md §3 step PX)
        float e[BATCH];
        bool any = false;
#pragma unroll
        for (int j = 0; j < BATCH; j++) {
            e[j] = 0.f;
            if (!done) {
                const float4 a = sm.rec0[buf][j];  // mx, my, r, o  (r = -1 for padding)
                const float dx = __fsub_rn(px, a.x), dy = __fsub_rn(py, a.y);
                if (fabsf(dx) <= a.z && fabsf(dy) <= a.z) {
                    tests++;
                    const float4 b = sm.rec1[buf][j];  // qa, qb, qc, ycut
                    const float q = __fmaf_rn(dx, __fmaf_rn(b.x, dx, __fmul_rn(b.y, dy)),
                                              __fmul_rn(__fmul_rn(b.z, dy), dy));
                    if (!(q > 0.f) && q >= b.w) {
                        const float al = fminf(K_ACLAMP, __fmul_rn(a.w, exp2_spec(q)));
                        if (al >= K_AMIN) {
                            const float Tn = __fmul_rn(T, __fsub_rn(1.0f, al));
                            if (Tn < K_TMIN) {
                                done = true;
                            } else {
                                e[j] = __fmul_rn(al, T);
                                T = Tn;
                                cnt++;
                                any = true;
                            }
                        }
                    }
                }
            }
        }

        if (!overflow) {
            // ---- per (warp, region group) transpose-reduction, then shared accumulation
            if (__any_sync(FULL, any)) {
                float zsum = 0.f;
                if (grp == FULL) {
                    const float v = transpose_reduce<false>(e, true, lane);
                    if (v != 0.f) smem_add(&sm.acc[buf][slot * BATCH + lane], v);
                    zsum = v;
                } else {
                    unsigned todo = FULL;
                    while (todo) {
                        const int l = __ffs(todo) - 1;
                        const unsigned g2 = __shfl_sync(FULL, grp, l);
                        const int q = __shfl_sync(FULL, slot, l);
                        todo &= ~g2;
                        const float v = transpose_reduce<true>(e, (g2 >> lane) & 1u, lane);
                        if (v != 0.f) smem_add(&sm.acc[buf][q * BATCH + lane], v);
                        zsum += v;
                    }
                }
                if (zsum != 0.f) smem_add(&sm.accZ[buf][lane], zsum);
            }
            __syncthreads();  // B1
            // ---- flush: S reds per (slot, Gaussian) into W, one per Gaussian into Z
            const int nitems = nslot * BATCH * S;
            for (int i = t; i < nitems; i += TILE_PIX) {
                const int q = i / (BATCH * S);
                const int rem = i - q * (BATCH * S);
                const int j = rem / S, s = rem - j * S;
                const float v = sm.acc[buf][q * BATCH + j];
                const uint32_t a = sm.slot_atom[q][s];
                if (v > 0.f && a != NONE)
                    atomicAdd(Wm + (int64_t)sm.gid[buf][j] * L + a, __fmul_rn(sm.slot_coef[q][s], v));
            }
            if (t < BATCH) {
                const float z = sm.accZ[buf][t];
                if (z > 0.f) atomicAdd(p.Z + sm.gid[buf][t], z);
            }
            // zero the other accumulator buffer (last flushed one batch ago)
            for (int i = t; i < nslot * BATCH; i += TILE_PIX) sm.acc[buf ^ 1][i] = 0.f;
            if (t < BATCH) sm.accZ[buf ^ 1][t] = 0.f;
        } else {
            // ---- fallback: per-pixel reductions straight from the code table
            if (any) {
                const bool coded = key != KEY_NONE;
                const int64_t row = (p.code_row0 + (int64_t)(coded ? key : 0)) * S;
#pragma unroll 1
                for (int j = 0; j < BATCH; j++) {
                    if (e[j] > 0.f) {
                        const uint32_t g = sm.gid[buf][j];
                        atomicAdd(p.Z + g, e[j]);
                        if (coded) {
                            for (int s = 0; s < S; s++) {
                                const uint32_t a = __ldg(p.code_atoms + row + s);
                                if (a != NONE)
                                    atomicAdd(Wm + (int64_t)g * L + a, __fmul_rn(__ldg(p.code_coefs + row + s), e[j]));
                            }
                        }
                    }
                }
            }
        }
        // stage the prefetched records for the next batch
        if (warp == 0) {
            sm.gid[buf ^ 1][lane] = ng;
            sm.rec0[buf ^ 1][lane] = nr0;
            sm.rec1[buf ^ 1][lane] = nr1;
        }
        if (__syncthreads_count(!done) == 0) break;  // B2
        (void)n;
    }

    // contributions (terms of Eq. 5's sum)
    unsigned c = __reduce_add_sync(FULL, cnt);
    unsigned ts = __reduce_add_sync(FULL, tests);
    if (lane == 0 && c) atomicAdd(&sm.contrib, (unsigned long long)c);
    if (lane == 0 && ts) atomicAdd(&sm.tests, (unsigned long long)ts);
    __syncthreads();
    if (t == 0) {
        if (sm.contrib) {
            atomicAdd(p.contrib_ctr, sm.contrib);
            if (p.contrib_out) atomicAdd(reinterpret_cast<unsigned long long*>(p.contrib_out), sm.contrib);
        }
        if (sm.tests) atomicAdd(p.support_ctr, sm.tests);
    }
}

}  // namespace

void launch_raster(const RasterParams& p, cudaStream_t s) {
    const int ntiles = p.tiles_x * p.tiles_y;
    if (ntiles <= 0) return;
    raster_aggregate_kernel<<<ntiles, TILE_PIX, 0, s>>>(p);
}

}  // namespace scoup
