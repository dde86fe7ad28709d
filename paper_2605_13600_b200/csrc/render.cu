// render.cu -- sparse coefficient rendering (Eq. 7).
//
//   W_hat_v(p) = sum_{i in N_{v,p}} w_hat_i e_i(v,p)
//
// with the K-sparse stored codes w_hat_i (Eq. 6) and the same fragment weights e_i(v,p) as the
// uplift -- the same depth chunks, candidate lists and DESIGN.md §3 per-pixel sequence
// (pixel_fragment), so every e is bit-identical to the CPU oracle's.  One CTA of 256 threads per
// (view, 16x16 tile), one pixel per thread; each pixel accumulates its dense L-vector in a padded
// shared-memory row (stride L + 1: the 32 lanes' read-modify-writes of one atom hit 32 banks).
// A batch record's K (atom, coef) pairs are staged in shared memory with repeated atoms merged
// and empty / padding slots pointed at the row's pad column, so a contribution's K updates are
// independent: their loads issue back to back (8 at a time) instead of as a serial
// load-add-store chain.  The rows are carried between depth chunks through the output buffer
// itself: chunk 0 writes them (zeros for tiles nothing reaches), later chunks add to them; the
// row I/O moves float4s along tile rows, which are contiguous in the [H, W, L] output.
#include "internal.cuh"

namespace scoup {

namespace {

constexpr unsigned FULL = 0xffffffffu;
constexpr int QCAP = 512;  // candidate ring (power of two >= 256 + BATCH)
constexpr int NWARP = TILE_PIX / 32;
constexpr int MAX_RK = 32;  // stored code length K
constexpr int KG = 8;       // code slots updated per independent group

struct RRing {
    // pair-interleaved (mx, mx', my, my'), (r, r', o, o'), (qa, qa', qb, qb'), (qc, qc', ycut,
    // ycut') of records 2i, 2i+1, as in the uplift kernel (paired-FP32 evaluation)
    float4 p0[(QCAP + BATCH) / 2];
    float4 p1[(QCAP + BATCH) / 2];
    float4 p2[(QCAP + BATCH) / 2];
    float4 p3[(QCAP + BATCH) / 2];
    float4 q2[QCAP + BATCH];  // (support-box half-extents x, y, Gaussian id, sy)
    float4 q3[QCAP + BATCH];  // band_relevant parameters
};

struct __align__(16) RSmem {
    RRing r;
    __align__(16) uint32_t code_a[BATCH][MAX_RK];  // the batch records' stored codes: row column (pad: L)
    __align__(16) float code_c[BATCH][MAX_RK];     //   and coefficient (merged over repeats; pad: 0)
    int wcnt[NWARP];
    // followed by the per-pixel accumulators: float acc[TILE_PIX][L + 1] (dynamic)
};

// Move a tile's pixel rows between shared memory (row of the pixel's thread, stride L + 1) and
// the view's [H, W, L] output: i enumerates (tile row, column, 4-float group) so a tile row's
// 16 L floats are one contiguous run in global memory.  i / L4 in fp32: (i + 0.5) / L4 is at
// least 0.5 / L4 >= 1/64 from an integer and i < 2^13, so the truncation is exact.
template <bool OUT>
__device__ __forceinline__ void row_io(float* acc_base, float* out_view, int L, int tx, int ty, int Wd, int Hd,
                                       int t) {
    const int LP = L + 1;
    const int vw = (L & 3) == 0 ? 4 : 1;  // float4 groups when L % 4 == 0
    const int LG = L / vw;
    const float inv = 1.0f / (float)LG;
    for (int i = t; i < TILE_PIX * LG; i += TILE_PIX) {
        const int q = (int)(((float)i + 0.5f) * inv);  // pixel in the tile, row-major
        const int lg = i - q * LG;
        const int r = q >> 4, xx = q & 15;
        const int gx = tx * TILE + xx, gy = ty * TILE + r;
        if (gx >= Wd || gy >= Hd) continue;
        // thread of pixel (xx, r): 8x4 warp blocks, lanes row-major inside
        const int th = ((xx >> 3) + 2 * (r >> 2)) * 32 + (xx & 7) + 8 * (r & 3);
        float* srow = acc_base + th * LP + lg * vw;
        float* grow = out_view + ((int64_t)gy * Wd + gx) * L + lg * vw;
        if (vw == 4) {
            if (OUT) {
                *reinterpret_cast<float4*>(grow) = make_float4(srow[0], srow[1], srow[2], srow[3]);
            } else {
                const float4 g4 = *reinterpret_cast<const float4*>(grow);
                srow[0] = g4.x; srow[1] = g4.y; srow[2] = g4.z; srow[3] = g4.w;
            }
        } else {
            if (OUT) *grow = *srow;
            else *srow = *grow;
        }
    }
}

__global__ void __launch_bounds__(TILE_PIX, 1) render_kernel(const RasterParams p) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    RSmem& sm = *reinterpret_cast<RSmem*>(smem_raw);
    float* const acc_base = reinterpret_cast<float*>(smem_raw + sizeof(RSmem));
    const int L = p.L, LP = L + 1, rK = p.rK;
    const int ntiles = p.bn.tiles_x * p.bn.tiles_y;
    const int view = blockIdx.x / ntiles, tile = blockIdx.x - view * ntiles;
    const int tx = tile % p.bn.tiles_x, ty = tile / p.bn.tiles_x;
    const int64_t gtile = (int64_t)view * ntiles + tile;
    if (p.chunk > 0 && !p.tile_live[gtile]) return;
    const int bin = ((ty * TILE) >> p.bn.bshy) * p.bn.bins_x + ((tx * TILE) >> p.bn.bshx);
    const uint2 range = p.ranges[view * p.bn.nbins() + bin];
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const int wx0 = tx * TILE + 8 * (warp & 1), wy0 = ty * TILE + 4 * (warp >> 1);
    const int x = wx0 + (lane & 7), y = wy0 + (lane >> 3);
    const int Wd = p.width, Hd = p.height;
    const bool inside = x < Wd && y < Hd;
    float* Tpix = p.Tstate + (int64_t)view * Wd * Hd + (int64_t)y * Wd + x;
    float* out_tile = p.r_out + ((p.r_view0 + view) * (int64_t)Hd * Wd) * L;  // this view's [H, W, L]
    float* acc = acc_base + (int64_t)t * LP;                                  // my pixel's row

    // the tile's rows: zero (chunk 0) or the partial sums of the earlier chunks
    if (p.chunk == 0) {
        for (int i = t; i < TILE_PIX * LP; i += TILE_PIX) acc_base[i] = 0.f;
    } else {
        row_io<false>(acc_base, out_tile, L, tx, ty, Wd, Hd, t);
    }
    const bool empty = range.x >= range.y;
    float T = !inside ? 0.0f : (p.chunk == 0 ? 1.0f : *Tpix);

    const float TX0 = (float)(tx * TILE) + 0.5f, TY0 = (float)(ty * TILE) + 0.5f;
    const float TX1 = (float)(min(tx * TILE + TILE, Wd) - 1) + 0.5f;
    const float TY1 = (float)(min(ty * TILE + TILE, Hd) - 1) + 0.5f;
    const float WX0 = (float)wx0 + 0.5f, WY0 = (float)wy0 + 0.5f;
    const float WX1 = (float)(min(wx0 + 8, Wd) - 1) + 0.5f, WY1 = (float)(min(wy0 + 4, Hd) - 1) + 0.5f;
    const float px = __fadd_rn((float)x, 0.5f), py = __fadd_rn((float)y, 0.5f);
    const unsigned lanemask_lt = (1u << lane) - 1u;
    float* const pf0 = reinterpret_cast<float*>(sm.r.p0);
    float* const pf1 = reinterpret_cast<float*>(sm.r.p1);
    float* const pf2 = reinterpret_cast<float*>(sm.r.p2);
    float* const pf3 = reinterpret_cast<float*>(sm.r.p3);
    auto put_pair_rec = [&](uint32_t pos, const float4& r0, const float4& r1) {
        const uint32_t b = (pos >> 1) * 4 + (pos & 1);
        pf0[b] = r0.x; pf0[b + 2] = r0.y; pf1[b] = r0.z; pf1[b + 2] = r0.w;
        pf2[b] = r1.x; pf2[b + 2] = r1.y; pf3[b] = r1.z; pf3[b + 2] = r1.w;
    };
    auto get_rec0 = [&](uint32_t pos) {
        const uint32_t b = (pos >> 1) * 4 + (pos & 1);
        return make_float4(pf0[b], pf0[b + 2], pf1[b], pf1[b + 2]);
    };
    float4* const q2 = sm.r.q2;
    float4* const q3 = sm.r.q3;
    __syncthreads();

    uint32_t cursor = range.x, q_head = 0, q_count = 0;
    while (!empty) {
        // ---- refill (as the uplift kernel: tile test, stable compaction into the ring)
        while (q_count < (uint32_t)BATCH && cursor < range.y) {
            const uint32_t idx = cursor + t;
            bool accp = false;
            float4 r0 = make_float4(0.f, 0.f, -1.f, 0.f), r1 = make_float4(0.f, 0.f, 0.f, 0.f);
            float4 r2 = make_float4(-1.f, -1.f, 0.f, 0.f), r3 = make_float4(0.f, 0.f, 0.f, -1.f);
            if (idx < range.y) {
                const uint32_t e = __ldg(p.eval + idx);
                r0 = __ldg(p.rec0 + e);
                r2 = __ldg(p.rec2 + e);
                r3 = __ldg(p.rec3 + e);
                accp = band_relevant(r0, r2, r3, TX0, TX1, TY0, TY1);
                if (accp) r1 = __ldg(p.rec1 + e);
            }
            const unsigned bal = __ballot_sync(FULL, accp);
            if (lane == 0) sm.wcnt[warp] = __popc(bal);
            __syncthreads();
            uint32_t off = 0, tot = 0;
#pragma unroll
            for (int w = 0; w < NWARP; w++) {
                const uint32_t c = (uint32_t)sm.wcnt[w];
                off += (w < warp) ? c : 0u;
                tot += c;
            }
            if (accp) {
                const uint32_t pos = (q_head + q_count + off + __popc(bal & lanemask_lt)) & (QCAP - 1);
                put_pair_rec(pos, r0, r1); q2[pos] = r2; q3[pos] = r3;
                if (pos < (uint32_t)BATCH) {
                    put_pair_rec(pos + QCAP, r0, r1); q2[pos + QCAP] = r2; q3[pos + QCAP] = r3;
                }
            }
            q_count += tot;
            cursor += TILE_PIX;
            __syncthreads();
        }
        if (q_count == 0) break;
        const uint32_t n = min((uint32_t)BATCH, q_count);
        // ---- stage the batch records' stored codes (Eq. 6 output): K rounded up to a multiple
        //      of KG, empty / out-of-range slots -> the pad column L, repeated atoms merged into
        //      their first slot so the slots of one record address distinct columns
        const int rKp = (rK + KG - 1) / KG * KG;
        for (int i = t; i < BATCH * rKp; i += TILE_PIX) {
            const int j = i / rKp, k = i - j * rKp;
            uint32_t a = NONE;
            float c = 0.f;
            if ((uint32_t)j < n && k < rK) {
                const uint32_t g = __float_as_uint(q2[(q_head + j) & (QCAP - 1)].z);
                a = __ldg(p.r_atoms + (int64_t)g * rK + k);
                c = __ldg(p.r_coefs + (int64_t)g * rK + k);
                if ((a != NONE && a >= (uint32_t)L) || !isfinite(c)) {
                    latch_error(p.err, ERR_CODE, (long long)g * rK + k);
                    a = NONE;
                }
            }
            sm.code_a[j][k] = a;
            sm.code_c[j][k] = c;
        }
        __syncthreads();
        constexpr int SPT = BATCH * MAX_RK / TILE_PIX;  // slots per thread
        float cm[SPT];
        uint32_t am[SPT];
#pragma unroll
        for (int u = 0; u < SPT; u++) {
            const int i = t + u * TILE_PIX;
            am[u] = (uint32_t)L;
            cm[u] = 0.f;
            if (i < BATCH * rKp) {
                const int j = i / rKp, k = i - j * rKp;
                const uint32_t a = sm.code_a[j][k];
                bool first = a != NONE;
                for (int k2 = 0; k2 < k && first; k2++) first = sm.code_a[j][k2] != a;
                if (first) {
                    float c = sm.code_c[j][k];
                    for (int k2 = k + 1; k2 < rK; k2++)
                        if (sm.code_a[j][k2] == a) c = __fadd_rn(c, sm.code_c[j][k2]);
                    am[u] = a;
                    cm[u] = c;
                }
            }
        }
        __syncthreads();
#pragma unroll
        for (int u = 0; u < SPT; u++) {
            const int i = t + u * TILE_PIX;
            if (i < BATCH * rKp) {
                const int j = i / rKp, k = i - j * rKp;
                sm.code_a[j][k] = am[u];
                sm.code_c[j][k] = cm[u];
            }
        }
        __syncthreads();
        // ---- per-warp mask, then the records in depth order; each contribution adds
        //      coef * e to the pixel's row at its atoms (Eq. 7)
        const bool warp_done = __all_sync(FULL, T == 0.f);
        bool rel = false;
        if (!warp_done && (uint32_t)lane < n)
            rel = band_relevant(get_rec0(q_head + lane), q2[q_head + lane], q3[q_head + lane], WX0, WX1, WY0, WY1);
        const unsigned mask = __ballot_sync(FULL, rel);
        const ulonglong2* b0 = reinterpret_cast<const ulonglong2*>(sm.r.p0) + (q_head >> 1);
        const ulonglong2* b1 = reinterpret_cast<const ulonglong2*>(sm.r.p1) + (q_head >> 1);
        const ulonglong2* b2 = reinterpret_cast<const ulonglong2*>(sm.r.p2) + (q_head >> 1);
        const ulonglong2* b3 = reinterpret_cast<const ulonglong2*>(sm.r.p3) + (q_head >> 1);
        for (int j2 = 0; j2 < BATCH; j2 += 2) {
            const unsigned pm = (mask >> j2) & 3u;
            if (!pm) continue;  // warp-uniform
            // the T-independent part of DESIGN.md §3 PX for records j2, j2+1 in paired FP32
            const ulonglong2 A0 = b0[j2 >> 1], A1 = b1[j2 >> 1], A2 = b2[j2 >> 1], A3 = b3[j2 >> 1];
            const f2 dx2 = f2_rsub(A0.x, px), dy2 = f2_rsub(A0.y, py);
            const f2 q2v = f2_fma(dx2, f2_fma(A2.x, dx2, f2_mul(A2.y, dy2)), f2_mul(f2_mul(A3.x, dy2), dy2));
            float op0, op1, dxs[2], dys[2], qs[2], rs[2], ys[2];
            f2_split(f2_mul(A1.y, exp2_spec2(q2v)), op0, op1);
            const float al2[2] = {fminf(K_ACLAMP, op0), fminf(K_ACLAMP, op1)};
            float om[2];
            f2_split(f2_rsub(f2_pack(al2[0], al2[1]), 1.0f), om[0], om[1]);
            f2_split(dx2, dxs[0], dxs[1]);
            f2_split(dy2, dys[0], dys[1]);
            f2_split(q2v, qs[0], qs[1]);
            f2_split(A1.x, rs[0], rs[1]);
            f2_split(A3.y, ys[0], ys[1]);
#pragma unroll
            for (int h = 0; h < 2; h++) {
            if (!((pm >> h) & 1u)) continue;  // warp-uniform
            const int j = j2 + h;
            const bool sq = fabsf(dxs[h]) <= rs[h] && fabsf(dys[h]) <= rs[h];
            const float al = al2[h];
            const float Tn = __fmul_rn(T, om[h]);
            const bool pass = sq && !(qs[h] > 0.f) && qs[h] >= ys[h] && al >= K_AMIN;
            const bool con = pass && !(Tn < K_TMIN);
            const float e = con ? __fmul_rn(al, T) : 0.f;
            T = con ? Tn : (pass ? 0.f : T);
            if (con) {
                for (int k0 = 0; k0 < rKp; k0 += KG) {
                    const uint4 a0 = *reinterpret_cast<const uint4*>(&sm.code_a[j][k0]);
                    const uint4 a1 = *reinterpret_cast<const uint4*>(&sm.code_a[j][k0 + 4]);
                    const uint32_t a[KG] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
                    const float4 c0 = *reinterpret_cast<const float4*>(&sm.code_c[j][k0]);
                    const float4 c1 = *reinterpret_cast<const float4*>(&sm.code_c[j][k0 + 4]);
                    const float c[KG] = {c0.x, c0.y, c0.z, c0.w, c1.x, c1.y, c1.z, c1.w};
                    float v[KG];
#pragma unroll
                    for (int k = 0; k < KG; k++) v[k] = acc[a[k]];  // distinct columns (or the pad)
#pragma unroll
                    for (int k = 0; k < KG; k++) acc[a[k]] = __fmaf_rn(c[k], e, v[k]);
                }
            }
            }
        }
        q_head = (q_head + n) & (QCAP - 1);
        q_count -= n;
        if (__syncthreads_count(T > 0.f) == 0) break;
    }
    __syncthreads();
    // ---- rows out, state for the next chunk
    row_io<true>(acc_base, out_tile, L, tx, ty, Wd, Hd, t);
    if (inside) *Tpix = T;
    const int live = __syncthreads_count(T > 0.f);
    if (t == 0) p.tile_live[gtile] = live > 0 ? 1 : 0;
}

}  // namespace

size_t render_smem_bytes(int L) { return sizeof(RSmem) + (size_t)TILE_PIX * (L + 1) * sizeof(float); }

void launch_render(const RasterParams& p, cudaStream_t s) {
    const int ntiles = p.bn.tiles_x * p.bn.tiles_y * p.nviews;
    if (ntiles <= 0) return;
    const size_t smem = render_smem_bytes(p.L);
    static size_t attr = 0;
    if (smem > attr) {
        cudaFuncSetAttribute(render_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        attr = smem;
    }
    render_kernel<<<ntiles, TILE_PIX, smem, s>>>(p);
}

}  // namespace scoup
