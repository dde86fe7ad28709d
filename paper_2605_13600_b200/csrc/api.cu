// api.cu -- C ABI (include/scoup.h) and host orchestration of the sm_100a path.
//
// Per view (Algorithm 1 lines 5-12):
//   stage 1  preprocess (EWA, culls, support rect)  ->  depth sort (CUB radix, stable, so
//            equal depths keep index order)  ->  scan of tile counts in depth
//            order  ->  entry total copied to pinned host memory
//   stage 2  emit (Gaussian, tile) entries in depth order  ->  stable radix sort on the tile
//            id  ->  per-tile ranges  ->  fused rasterise-and-aggregate kernel
// Stage 2 needs the entry total on the host (CUB takes host-side sizes), so two view
// contexts on two streams are software-pipelined: while the host waits for view v's total,
// the GPU runs view v-1's raster.
// finalize_topk runs Eq. 6 on the requested rows.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/iterator/transform_input_iterator.cuh>

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/scoup.h"
#include "internal.cuh"

using namespace scoup;

namespace {

thread_local std::string g_last_error;

scoup_status fail(scoup_status st, const std::string& msg) {
    g_last_error = msg;
    return st;
}

struct CudaError {
    cudaError_t err;
    std::string where;
};

#define CK(expr)                                                    \
    do {                                                            \
        cudaError_t _e = (expr);                                    \
        if (_e != cudaSuccess) throw CudaError{_e, #expr};          \
    } while (0)

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev) cudaSetDevice(dev);
    }
    ~DeviceGuard() {
        int cur = -1;
        cudaGetDevice(&cur);
        if (prev >= 0 && cur != prev) cudaSetDevice(prev);
    }
};

bool is_device_ptr(const void* p) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

// Device memory is stream-ordered (cudaMallocAsync on the stream that uses it) from the
// device's default memory pool, whose release threshold init raises so that freed blocks stay
// cached: creating and freeing handles per scene costs no cudaMalloc/cudaFree round trips.
template <typename T>
void dalloc(T** ptr, size_t count, cudaStream_t s) {
    *ptr = nullptr;
    CK(cudaMallocAsync((void**)ptr, std::max<size_t>(count, 1) * sizeof(T), s));
}

void dfree(void* p, cudaStream_t s) {
    if (p) cudaFreeAsync(p, s);
}

template <typename T>
void grow(T** ptr, size_t* cap, size_t need, cudaStream_t s, double slack = 1.25) {
    if (need <= *cap && *ptr) return;
    size_t n = std::max<size_t>(need, (size_t)((double)need * slack));
    if (*ptr) CK(cudaFreeAsync(*ptr, s));
    *ptr = nullptr;
    *cap = 0;
    dalloc(ptr, n, s);
    *cap = n;
}

// One pipeline context: the buffers of one view batch and the stream it runs on.  Two
// contexts alternate so that batch b+1's projection and depth sort overlap batch b's raster.
struct Ctx {
    cudaStream_t s = nullptr;
    cudaEvent_t ev_total = nullptr;
    ViewBuffers vb{};
    size_t g_cap = 0, e_cap = 0, t_cap = 0;
    void* cub_tmp = nullptr;
    size_t cub_cap = 0;
    uint64_t* h_total = nullptr;  // pinned [MAX_VB]: offsets at the end of each view
    uint32_t* ids_stage = nullptr;
    size_t ids_cap = 0;
    // launch state of the batch in flight (stage 1 done, stage 2 pending)
    int v0 = 0, nv = 0;
    int key_bits = 32;
    const uint32_t* ids_dev[MAX_VB] = {};
    // timing: ring of event sets (start/end of stage 1, binning start, raster start/end)
    struct EvSet { cudaEvent_t e[5]; bool pending; int views; };
    std::vector<EvSet> evs;
    int ev_next = 0;
    int ev_cur = -1;
};

}  // namespace

struct scoup_uplift {
    int device = 0;
    cudaStream_t stream = nullptr;
    int64_t G = 0, Npad = 0;
    int L = 0, K = 0;
    float* W = nullptr;
    float* Z = nullptr;
    bool own_wz = false;
    PackedGaussians pg{};
    int* d_err_code = nullptr;
    long long* d_err_index = nullptr;
    unsigned long long* d_stats = nullptr;  // views, contributions, entries, visible
    Ctx ctx[2];
    uint32_t* code_atoms = nullptr;
    float* code_coefs = nullptr;
    size_t code_cap = 0;
    uint32_t* code_atoms_in = nullptr;
    float* code_coefs_in = nullptr;
    int64_t host_entries = 0;
    cudaEvent_t ev_fork = nullptr, ev_join[2] = {nullptr, nullptr};
    bool latched = false;
    int sms = 148;
    // timing + launch accounting
    bool timing = false;
    double t_pre = 0, t_bin = 0, t_ras = 0, t_topk = 0;
    int64_t ras_launches = 0, views_timed = 0;
    cudaEvent_t topk_ev[2] = {nullptr, nullptr};
    bool topk_pending = false;
    int64_t kernel_launches = 0, cub_launches = 0;
    double bb[6] = {0, 0, 0, 0, 0, 0};  // box of the valid means (x0, y0, z0, x1, y1, z1)
};

namespace {

ErrorLatch latch_of(scoup_uplift* h) { return ErrorLatch{h->d_err_code, h->d_err_index}; }

scoup_status check_latched(scoup_uplift* h) {
    int code = 0;
    long long idx = 0;
    CK(cudaMemcpy(&code, h->d_err_code, sizeof(int), cudaMemcpyDeviceToHost));
    if (code == ERR_NONE) return SCOUP_OK;
    CK(cudaMemcpy(&idx, h->d_err_index, sizeof(long long), cudaMemcpyDeviceToHost));
    h->latched = true;
    if (code == ERR_DEPTHKEY)
        return fail(SCOUP_ECUDA, "internal error: depth code beyond the batch bound at batch index " + std::to_string(idx));
    const char* what = code == ERR_GAUSSIAN ? "non-finite or invalid Gaussian parameters at Gaussian index "
                       : code == ERR_REGION ? "region id >= num_regions at flat pixel index "
                                            : "invalid code slot (atom >= L or bad coefficient) at flat slot index ";
    return fail(SCOUP_EDATA, std::string("data error: ") + what + std::to_string(idx));
}

void ctx_init(Ctx& c) {
    CK(cudaStreamCreateWithFlags(&c.s, cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&c.ev_total, cudaEventDisableTiming));
    CK(cudaMallocHost((void**)&c.h_total, sizeof(uint64_t) * MAX_VB));
}

void ctx_free(Ctx& c, cudaStream_t s) {
    for (auto& es : c.evs)
        for (int k = 0; k < 5; k++) cudaEventDestroy(es.e[k]);
    c.evs.clear();
    ViewBuffers& b = c.vb;
    void* ptrs[] = {b.depth_key, b.depth_key_alt, b.dval, b.dval_sorted, b.tiles, b.offsets, b.rect,
                    b.rec0, b.rec1, b.rec2, b.totals, b.ekey, b.eval, b.ekey_alt, b.eval_alt, b.ranges, b.bin_count,
                    c.cub_tmp, c.ids_stage};
    for (void* p : ptrs) dfree(p, s);
    if (c.h_total) cudaFreeHost(c.h_total);
    if (c.ev_total) cudaEventDestroy(c.ev_total);
    if (c.s) cudaStreamDestroy(c.s);
    c = Ctx{};
}

// Per-(view, Gaussian) buffers for a batch of n = B*G elements.
void ctx_reserve_gaussians(Ctx& c, int64_t n) {
    if ((size_t)n <= c.g_cap && c.vb.depth_key) return;
    ViewBuffers& b = c.vb;
    n = std::max<int64_t>(n, 1);
#define RG(f) { dalloc(&b.f, (size_t)n, c.s); }
    if (b.depth_key) {
        void* ptrs[] = {b.depth_key, b.depth_key_alt, b.dval, b.dval_sorted, b.tiles, b.offsets, b.rect, b.rec0, b.rec1,
                        b.rec2};
        for (void* p : ptrs) dfree(p, c.s);
    }
    RG(depth_key) RG(depth_key_alt) RG(dval) RG(dval_sorted) RG(tiles) RG(offsets) RG(rect) RG(rec0) RG(rec1) RG(rec2)
#undef RG
    if (!b.totals) dalloc(&b.totals, MAX_VB, c.s);
    c.g_cap = (size_t)n;
}

void ctx_reserve_cub(Ctx& c, size_t bytes) { grow((char**)&c.cub_tmp, &c.cub_cap, bytes, c.s); }

bool rigid_ok(const float* M) {
    double R[3][3];
    for (int a = 0; a < 3; a++)
        for (int b = 0; b < 3; b++) R[a][b] = M[4 * a + b];
    for (int a = 0; a < 3; a++)
        for (int b = 0; b < 3; b++) {
            double d = 0;
            for (int k = 0; k < 3; k++) d += R[a][k] * R[b][k];
            if (std::fabs(d - (a == b ? 1.0 : 0.0)) > 1e-5) return false;
        }
    double det = R[0][0] * (R[1][1] * R[2][2] - R[1][2] * R[2][1]) - R[0][1] * (R[1][0] * R[2][2] - R[1][2] * R[2][0]) +
                 R[0][2] * (R[1][0] * R[2][1] - R[1][1] * R[2][0]);
    if (std::fabs(det - 1.0) > 1e-5) return false;
    for (int k = 0; k < 16; k++)
        if (!std::isfinite(M[k])) return false;
    return true;
}

Camera to_cam(const scoup_camera& c) {
    Camera k;
    k.fx = c.fx; k.fy = c.fy; k.cx = c.cx; k.cy = c.cy;
    k.width = c.width; k.height = c.height;
    for (int i = 0; i < 12; i++) k.P[i] = c.world_to_camera[i];
    return k;
}

int bits_for(uint32_t n) {
    int b = 1;
    while ((1u << b) < n && b < 32) b++;
    return b;
}

constexpr int EV_RING = 8;

void ev_accumulate(scoup_uplift* h, Ctx::EvSet& es) {
    if (!es.pending) return;
    CK(cudaEventSynchronize(es.e[4]));
    float a = 0, b = 0, c = 0;
    CK(cudaEventElapsedTime(&a, es.e[0], es.e[1]));
    CK(cudaEventElapsedTime(&b, es.e[2], es.e[3]));
    CK(cudaEventElapsedTime(&c, es.e[3], es.e[4]));
    h->t_pre += a;
    h->t_bin += b;
    h->t_ras += c;
    h->ras_launches++;
    h->views_timed += es.views;
    es.pending = false;
}

Ctx::EvSet* ev_begin(scoup_uplift* h, Ctx& c) {
    if (!h->timing) { c.ev_cur = -1; return nullptr; }
    if (c.evs.empty()) {
        c.evs.resize(EV_RING);
        for (auto& es : c.evs) {
            for (int k = 0; k < 5; k++) CK(cudaEventCreate(&es.e[k]));
            es.pending = false;
        }
    }
    c.ev_cur = c.ev_next;
    c.ev_next = (c.ev_next + 1) % EV_RING;
    Ctx::EvSet& es = c.evs[c.ev_cur];
    ev_accumulate(h, es);
    return &es;
}

Ctx::EvSet* ev_cur(Ctx& c) { return c.ev_cur >= 0 ? &c.evs[c.ev_cur] : nullptr; }

// Stage 1 of one view: preprocess, depth sort, scan -> total entries (async to pinned host).
// Bin size: the smallest power-of-two group of tiles (>= 64x64 px) whose bin count fits one
// 8-bit radix pass (<= 256 bins); very large images fall back to <= 1024 bins (2 passes).
Binning choose_binning(int Wd, int Hd) {
    Binning b;
    b.tiles_x = (Wd + TILE - 1) / TILE;
    b.tiles_y = (Hd + TILE - 1) / TILE;
    const int cand[][2] = {{6, 6}, {7, 6}, {7, 7}, {8, 7}, {8, 8}, {9, 8}, {9, 9}, {10, 9}, {10, 10}, {11, 10},
                           {11, 11}, {12, 11}, {12, 12}};
    for (int lim : {256, 1024}) {
        for (auto& c : cand) {
            int bx = (Wd + (1 << c[0]) - 1) >> c[0], by = (Hd + (1 << c[1]) - 1) >> c[1];
            if (bx * by <= lim) {
                b.bshx = c[0]; b.bshy = c[1]; b.bins_x = bx; b.bins_y = by;
                return b;
            }
        }
    }
    b.bshx = b.bshy = 12;
    b.bins_x = (Wd + 4095) >> 12;
    b.bins_y = (Hd + 4095) >> 12;
    return b;
}

// Depth-code width for a batch: visible keys are bits(t_z) - bits(0.2f) in [1, bits(bound) -
// bits(0.2f)], with `bound` an upper bound of t_z over the scene box for every camera of the
// batch (exact max of the linear map over the box's corners, fp64, padded).  The code must
// leave the all-ones value free for invisible Gaussians.
int depth_key_bits(const scoup_uplift* h, const Camera* cams, int n) {
    double zmax = 0.2;
    for (int v = 0; v < n; v++) {
        const float* P = cams[v].P;
        for (int corner = 0; corner < 8; corner++) {
            const double x = (corner & 1) ? h->bb[3] : h->bb[0], y = (corner & 2) ? h->bb[4] : h->bb[1],
                         z = (corner & 4) ? h->bb[5] : h->bb[2];
            zmax = std::max(zmax, (double)P[8] * x + (double)P[9] * y + (double)P[10] * z + (double)P[11]);
        }
    }
    const double bound = zmax * (1.0 + 1e-4) + 1e-4;
    if (!(bound < 3.0e38)) return 32;
    const float bf = (float)bound;
    uint32_t bbits, nbits;
    std::memcpy(&bbits, &bf, 4);
    const float nearf = 0.2f;
    std::memcpy(&nbits, &nearf, 4);
    const uint64_t need = (uint64_t)(bbits - nbits) + 2;  // largest visible code + the none code
    int k = 1;
    while (k < 32 && (1ull << k) < need) k++;
    return k;
}

// Stage 1 of a view batch: preprocess (all B views in one launch), one stable radix sort of
// the (view, depth) keys, scan of the bin counts in that order -> per-view entry totals
// (async to pinned host).
void stage1(scoup_uplift* h, Ctx& c, const Camera* cams, int nv, const Binning& bn) {
    const int64_t G = h->G;
    const int64_t n = (int64_t)nv * G;
    ViewBuffers& b = c.vb;
    CamBatch cb{};
    cb.n = nv;
    for (int v = 0; v < nv; v++) cb.cam[v] = cams[v];
    int vbits = 0;
    while ((1 << vbits) < nv) vbits++;
    const int kb = vbits == 0 ? 32 : c.key_bits;  // single view: full 32-bit code
    const int end_bit = vbits == 0 ? 32 : kb + vbits;
    Ctx::EvSet* es = ev_begin(h, c);
    if (es) { CK(cudaEventRecord(es->e[0], c.s)); es->views = nv; }
    launch_preprocess(h->pg, G, cb, bn, b, kb, h->d_stats + 3, latch_of(h), c.s);
    size_t need = 0;
    CK(cub::DeviceRadixSort::SortPairs(nullptr, need, b.depth_key, b.depth_key_alt, b.dval, b.dval_sorted, (int)n, 0,
                                       end_bit, c.s));
    size_t need2 = 0;
    CK(cub::DeviceScan::InclusiveSum(nullptr, need2, b.offsets, b.offsets, (int)n, c.s));
    ctx_reserve_cub(c, std::max(need, need2));
    CK(cub::DeviceRadixSort::SortPairs(c.cub_tmp, need, b.depth_key, b.depth_key_alt, b.dval, b.dval_sorted, (int)n,
                                       0, end_bit, c.s));
    launch_gather_scan_input(b.dval_sorted, b.tiles, b.offsets, n, c.s);
    CK(cub::DeviceScan::InclusiveSum(c.cub_tmp, need2, b.offsets, b.offsets, (int)n, c.s));
    launch_view_totals(b.offsets, G, nv, b.totals, c.s);
    CK(cudaMemcpyAsync(c.h_total, b.totals, sizeof(uint64_t) * nv, cudaMemcpyDeviceToHost, c.s));
    if (es) CK(cudaEventRecord(es->e[1], c.s));
    CK(cudaEventRecord(c.ev_total, c.s));
    h->kernel_launches += 3;
    h->cub_launches += 2;
}

// Stage 2 of a view batch: emit, bin sort, ranges, raster.  Needs stage 1's totals on the host.
scoup_status stage2(scoup_uplift* h, Ctx& c, const Camera* cams, const Binning& bn, const int64_t* code_row0,
                    const int32_t* num_regions, int S, long long* contrib_out, int64_t npx) {
    CK(cudaEventSynchronize(c.ev_total));
    const int nv = c.nv;
    const int64_t G = h->G;
    const int64_t n = (int64_t)nv * G;
    const uint64_t E = c.h_total[nv - 1];
    const int nbins = bn.nbins() * nv;
    ViewBuffers& b = c.vb;
    if (E >= (uint64_t)INT32_MAX)
        return fail(SCOUP_EUNSUPPORTED, "view batch produces " + std::to_string(E) + " bin entries (>= 2^31)");
    if ((size_t)nbins > c.t_cap || !b.ranges) {
        dfree(b.ranges, c.s);
        dfree(b.bin_count, c.s);
        dalloc(&b.ranges, nbins, c.s);
        dalloc(&b.bin_count, nbins, c.s);
        c.t_cap = nbins;
    }
    h->host_entries += (int64_t)E;
    Ctx::EvSet* es = ev_cur(c);
    if (es) CK(cudaEventRecord(es->e[2], c.s));
    if (E > 0) {
        if (E > c.e_cap || !b.ekey) {
            size_t ne = (size_t)((double)E * 1.25);
            void* ptrs[] = {b.ekey, b.eval, b.ekey_alt, b.eval_alt};
            for (void* p : ptrs) dfree(p, c.s);
            dalloc(&b.ekey, ne, c.s);
            dalloc(&b.eval, ne, c.s);
            dalloc(&b.ekey_alt, ne, c.s);
            dalloc(&b.eval_alt, ne, c.s);
            c.e_cap = ne;
        }
        CK(cudaMemsetAsync(b.bin_count, 0, sizeof(uint32_t) * nbins, c.s));
        launch_emit(b.dval_sorted, b.offsets, b.rect, bn, n, G, b.ekey, b.eval, b.bin_count, c.s);
        launch_ranges_from_counts(b.bin_count, nbins, b.ranges, c.s);
        const int nbits = bits_for((uint32_t)nbins);
        size_t need = 0;
        CK(cub::DeviceRadixSort::SortPairs(nullptr, need, b.ekey, b.ekey_alt, b.eval, b.eval_alt, (int)E, 0, nbits, c.s));
        ctx_reserve_cub(c, need);
        CK(cub::DeviceRadixSort::SortPairs(c.cub_tmp, need, b.ekey, b.ekey_alt, b.eval, b.eval_alt, (int)E, 0, nbits, c.s));
        RasterParams p{};
        p.nviews = nv;
        p.width = cams[0].width;
        p.height = cams[0].height;
        p.G = G;
        p.bn = bn;
        p.ranges = b.ranges;
        p.eval = b.eval_alt;
        p.rec0 = b.rec0;
        p.rec1 = b.rec1;
        p.rec2 = b.rec2;
        for (int v = 0; v < nv; v++) {
            const int u = c.v0 + v;
            p.region_ids[v] = c.ids_dev[v];
            p.code_row0[v] = code_row0[u];
            p.num_regions[v] = num_regions[u];
            p.pixel_base[v] = (long long)u * npx;
            p.contrib_out[v] = contrib_out ? contrib_out + u : nullptr;
        }
        p.code_atoms = h->code_atoms;
        p.code_coefs = h->code_coefs;
        p.S = S;
        p.L = h->L;
        p.W = h->W;
        p.Z = h->Z;
        p.contrib_ctr = h->d_stats + 1;
        p.support_ctr = h->d_stats + 4;
        p.err = latch_of(h);
        if (es) CK(cudaEventRecord(es->e[3], c.s));
        launch_raster(p, c.s);
        h->kernel_launches += 3;
        h->cub_launches += 1;
    } else if (es) {
        CK(cudaEventRecord(es->e[3], c.s));
    }
    if (es) {
        CK(cudaEventRecord(es->e[4], c.s));
        es->pending = true;
    }
    CK(cudaGetLastError());
    return SCOUP_OK;
}

__global__ void add_u64(unsigned long long* p, unsigned long long v) { atomicAdd(p, v); }

}  // namespace

extern "C" {

const char* scoup_last_error(void) { return g_last_error.c_str(); }

const char* scoup_version(void) { return "scoup-b200 0.1.0 (sm_100a)"; }

scoup_status scoup_uplift_init(int device, void* cuda_stream, int64_t num_gaussians, const float* means,
                               const float* scales, const float* rotations, const float* opacities, int32_t L,
                               int32_t K, float* W, float* Z, int64_t rows_padded, scoup_uplift** out) {
    g_last_error.clear();
    if (!out) return fail(SCOUP_EINVAL, "out is NULL");
    *out = nullptr;
    if (num_gaussians < 0) return fail(SCOUP_EINVAL, "num_gaussians < 0");
    if (num_gaussians > 0 && (!means || !scales || !rotations || !opacities))
        return fail(SCOUP_EINVAL, "Gaussian parameter pointer is NULL");
    if (K < 1) return fail(SCOUP_EINVAL, "K < 1");
    if (L < 1) return fail(SCOUP_EINVAL, "L < 1");
    if (K > L) return fail(SCOUP_EINVAL, "K > L (SPEC.md:291)");
    if (L > SCOUP_MAX_L || K > SCOUP_MAX_K) return fail(SCOUP_EUNSUPPORTED, "L or K beyond implementation limits");
    if (num_gaussians >= (int64_t)INT32_MAX) return fail(SCOUP_EUNSUPPORTED, "num_gaussians >= 2^31");
    if (rows_padded == 0) rows_padded = num_gaussians;
    if (rows_padded < num_gaussians) return fail(SCOUP_EINVAL, "rows_padded < num_gaussians");
    if ((W == nullptr) != (Z == nullptr)) return fail(SCOUP_EINVAL, "W and Z must both be given or both be NULL");
    scoup_uplift* h = new scoup_uplift();
    try {
        int ndev = 0;
        CK(cudaGetDeviceCount(&ndev));
        if (device < 0 || device >= ndev) {
            delete h;
            return fail(SCOUP_EINVAL, "bad device ordinal");
        }
        DeviceGuard dg(device);
        h->device = device;
        h->stream = (cudaStream_t)cuda_stream;
        h->G = num_gaussians;
        h->Npad = rows_padded;
        h->L = L;
        h->K = K;
        CK(cudaDeviceGetAttribute(&h->sms, cudaDevAttrMultiProcessorCount, device));
        {
            cudaMemPool_t pool;
            CK(cudaDeviceGetDefaultMemPool(&pool, device));
            uint64_t keep = UINT64_MAX;
            CK(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
        }
        cudaStream_t hs = h->stream;
        if (W) {
            h->W = W;
            h->Z = Z;
        } else {
            dalloc(&h->W, (size_t)std::max<int64_t>(1, rows_padded) * L, hs);
            dalloc(&h->Z, (size_t)std::max<int64_t>(1, rows_padded), hs);
            h->own_wz = true;
        }
        dalloc(&h->d_err_code, 1, hs);
        dalloc(&h->d_err_index, 1, hs);
        dalloc(&h->d_stats, 5, hs);
        CK(cudaMemsetAsync(h->d_err_code, 0, sizeof(int), h->stream));
        CK(cudaMemsetAsync(h->d_err_index, 0, sizeof(long long), h->stream));
        CK(cudaMemsetAsync(h->d_stats, 0, 5 * sizeof(unsigned long long), h->stream));
        CK(cudaMemsetAsync(h->W, 0, sizeof(float) * rows_padded * L, h->stream));
        CK(cudaMemsetAsync(h->Z, 0, sizeof(float) * rows_padded, h->stream));
        const int64_t G = std::max<int64_t>(1, num_gaussians);
        dalloc(&h->pg.a, G, hs);
        dalloc(&h->pg.b, G, hs);
        dalloc(&h->pg.c, G, hs);
        CK(cudaEventCreateWithFlags(&h->ev_fork, cudaEventDisableTiming));
        for (int i = 0; i < 2; i++) {
            CK(cudaEventCreateWithFlags(&h->ev_join[i], cudaEventDisableTiming));
            ctx_init(h->ctx[i]);
        }
        if (num_gaussians > 0) {
            const float* src[4] = {means, scales, rotations, opacities};
            const size_t cnt[4] = {3, 3, 4, 1};
            const float* dsrc[4];
            std::vector<float*> tmp;
            for (int k = 0; k < 4; k++) {
                if (is_device_ptr(src[k])) {
                    dsrc[k] = src[k];
                } else {
                    float* d = nullptr;
                    dalloc(&d, cnt[k] * num_gaussians, hs);
                    CK(cudaMemcpyAsync(d, src[k], sizeof(float) * cnt[k] * num_gaussians, cudaMemcpyHostToDevice,
                                       h->stream));
                    tmp.push_back(d);
                    dsrc[k] = d;
                }
            }
            launch_activate(dsrc[0], dsrc[1], dsrc[2], dsrc[3], num_gaussians, h->pg, latch_of(h), h->stream);
            CK(cudaGetLastError());
            // scene box (for the depth-code width of each view batch)
            int* dbox = nullptr;
            dalloc(&dbox, 6, hs);
            const int init_box[6] = {INT_MAX, INT_MAX, INT_MAX, INT_MIN, INT_MIN, INT_MIN};
            CK(cudaMemcpyAsync(dbox, init_box, sizeof(init_box), cudaMemcpyHostToDevice, hs));
            launch_bounds(h->pg, num_gaussians, dbox, hs);
            int box[6];
            CK(cudaMemcpyAsync(box, dbox, sizeof(box), cudaMemcpyDeviceToHost, hs));
            CK(cudaStreamSynchronize(hs));
            dfree(dbox, hs);
            for (int a = 0; a < 6; a++) {
                const int bits = box[a] >= 0 ? box[a] : box[a] ^ 0x7FFFFFFF;
                float f;
                std::memcpy(&f, &bits, 4);
                h->bb[a] = (box[0] > box[3]) ? 0.0 : (double)f;  // no valid Gaussian: empty box
            }
            // host inputs were copied (pageable copies complete before returning; pinned ones
            // are ordered before the frees below on the same stream)
            for (float* d : tmp) dfree(d, hs);
            if (!tmp.empty()) CK(cudaStreamSynchronize(hs));
        }
    } catch (const CudaError& e) {
        scoup_uplift_free(h);
        return fail(e.err == cudaErrorMemoryAllocation ? SCOUP_ENOMEM : SCOUP_ECUDA,
                    std::string("CUDA error in ") + e.where + ": " + cudaGetErrorString(e.err));
    }
    *out = h;
    return SCOUP_OK;
}

scoup_status scoup_uplift_add_views(scoup_uplift* h, int32_t num_views, const scoup_camera* cameras,
                                    const uint32_t* region_ids, const int64_t* code_row0, const int32_t* num_regions,
                                    const uint32_t* code_atoms, const float* code_coefs, int32_t S,
                                    int64_t* contributions_out) {
    g_last_error.clear();
    if (!h) return fail(SCOUP_EINVAL, "handle is NULL");
    if (h->latched) return fail(SCOUP_ESTATE, "a latched data error is pending; call scoup_uplift_reset");
    if (num_views < 0) return fail(SCOUP_EINVAL, "num_views < 0");
    if (num_views == 0) return SCOUP_OK;
    if (!cameras || !region_ids || !code_row0 || !num_regions || !code_atoms || !code_coefs)
        return fail(SCOUP_EINVAL, "NULL argument");
    if (S < 1) return fail(SCOUP_EINVAL, "S < 1");
    if (S > SCOUP_MAX_S) return fail(SCOUP_EUNSUPPORTED, "S > SCOUP_MAX_S");
    const int Wd = cameras[0].width, Hd = cameras[0].height;
    int64_t rows = 0;
    for (int v = 0; v < num_views; v++) {
        const scoup_camera& c = cameras[v];
        if (c.width != Wd || c.height != Hd) return fail(SCOUP_EINVAL, "cameras of one call must share width/height");
        if (c.width <= 0 || c.height <= 0) return fail(SCOUP_EINVAL, "camera width/height <= 0");
        if (!(c.fx > 0.f) || !(c.fy > 0.f) || !std::isfinite(c.fx) || !std::isfinite(c.fy) || !std::isfinite(c.cx) ||
            !std::isfinite(c.cy))
            return fail(SCOUP_EINVAL, "camera " + std::to_string(v) + ": bad intrinsics");
        if (!rigid_ok(c.world_to_camera))
            return fail(SCOUP_EDATA, "camera " + std::to_string(v) + ": world_to_camera is not rigid (1e-5)");
        if (code_row0[v] < 0 || num_regions[v] < 0) return fail(SCOUP_EINVAL, "negative code_row0 / num_regions");
        rows = std::max<int64_t>(rows, code_row0[v] + num_regions[v]);
    }
    if ((int64_t)Wd * Hd >= (int64_t)INT32_MAX) return fail(SCOUP_EUNSUPPORTED, "image too large");
    if (h->G == 0) return SCOUP_OK;
    const Binning bn = choose_binning(Wd, Hd);
    const int64_t npx = (int64_t)Wd * Hd;
    try {
        DeviceGuard dg(h->device);
        // ---- codes: copy (if host) + validate + truncate (Algorithm 1 per-pixel TopK)
        if (rows > 0) {
            const size_t nslots = (size_t)(rows * S);
            if (nslots > h->code_cap) {
                size_t cap = (size_t)((double)nslots * 1.25);
                dfree(h->code_atoms, h->stream);
                dfree(h->code_coefs, h->stream);
                dfree(h->code_atoms_in, h->stream);
                dfree(h->code_coefs_in, h->stream);
                h->code_cap = 0;
                dalloc(&h->code_atoms, cap, h->stream);
                dalloc(&h->code_coefs, cap, h->stream);
                dalloc(&h->code_atoms_in, cap, h->stream);
                dalloc(&h->code_coefs_in, cap, h->stream);
                h->code_cap = cap;
            }
            const uint32_t* ain = code_atoms;
            const float* cin = code_coefs;
            if (!is_device_ptr(code_atoms) || !is_device_ptr(code_coefs)) {
                CK(cudaMemcpyAsync(h->code_atoms_in, code_atoms, sizeof(uint32_t) * nslots, cudaMemcpyDefault, h->stream));
                CK(cudaMemcpyAsync(h->code_coefs_in, code_coefs, sizeof(float) * nslots, cudaMemcpyDefault, h->stream));
                ain = h->code_atoms_in;
                cin = h->code_coefs_in;
            }
            launch_ingest_codes(ain, cin, rows, S, h->K, h->L, h->code_atoms, h->code_coefs, latch_of(h), h->stream);
        }
        const bool ids_on_device = is_device_ptr(region_ids);
        // ---- view batches: B views per pass (bounded by the bin-table size)
        const int B = std::max(1, std::min(MAX_VB, std::min(MAX_BINS / bn.nbins(), (int)num_views)));
        // ---- fork the two pipeline contexts off the caller's stream
        CK(cudaEventRecord(h->ev_fork, h->stream));
        for (int i = 0; i < 2; i++) {
            CK(cudaStreamWaitEvent(h->ctx[i].s, h->ev_fork, 0));
            ctx_reserve_gaussians(h->ctx[i], (int64_t)B * h->G);
        }
        std::vector<Camera> cams(num_views);
        for (int v = 0; v < num_views; v++) cams[v] = to_cam(cameras[v]);
        const int nbatch = (num_views + B - 1) / B;
        scoup_status st = SCOUP_OK;
        for (int bi = 0; bi <= nbatch && st == SCOUP_OK; bi++) {
            if (bi < nbatch) {
                Ctx& c = h->ctx[bi & 1];
                c.v0 = bi * B;
                c.nv = std::min(B, num_views - c.v0);
                c.key_bits = depth_key_bits(h, &cams[c.v0], c.nv);
                if (!ids_on_device) grow(&c.ids_stage, &c.ids_cap, (size_t)(B * npx), c.s, 1.0);
                for (int v = 0; v < c.nv; v++) {
                    const int u = c.v0 + v;
                    if (ids_on_device) {
                        c.ids_dev[v] = region_ids + (int64_t)u * npx;
                    } else {
                        CK(cudaMemcpyAsync(c.ids_stage + (int64_t)v * npx, region_ids + (int64_t)u * npx,
                                           sizeof(uint32_t) * npx, cudaMemcpyHostToDevice, c.s));
                        c.ids_dev[v] = c.ids_stage + (int64_t)v * npx;
                    }
                }
                stage1(h, c, &cams[c.v0], c.nv, bn);
            }
            if (bi > 0) {
                Ctx& c = h->ctx[(bi - 1) & 1];
                st = stage2(h, c, &cams[c.v0], bn, code_row0, num_regions, S, (long long*)contributions_out, npx);
            }
        }
        // ---- join back into the caller's stream
        for (int i = 0; i < 2; i++) {
            CK(cudaEventRecord(h->ev_join[i], h->ctx[i].s));
            CK(cudaStreamWaitEvent(h->stream, h->ev_join[i], 0));
        }
        add_u64<<<1, 1, 0, h->stream>>>(h->d_stats + 0, (unsigned long long)num_views);
        h->kernel_launches += 1 + (rows > 0 ? 1 : 0);
        CK(cudaGetLastError());
        if (st != SCOUP_OK) return st;
    } catch (const CudaError& e) {
        return fail(e.err == cudaErrorMemoryAllocation ? SCOUP_ENOMEM : SCOUP_ECUDA,
                    std::string("CUDA error in ") + e.where + ": " + cudaGetErrorString(e.err));
    }
    return SCOUP_OK;
}

scoup_status scoup_uplift_finalize_topk(scoup_uplift* h, int64_t first_row, int64_t num_rows, const float* W_rows,
                                        const float* Z_rows, uint32_t* out_atoms, float* out_coefs) {
    g_last_error.clear();
    (void)Z_rows;
    if (!h) return fail(SCOUP_EINVAL, "handle is NULL");
    if (first_row < 0 || num_rows < 0) return fail(SCOUP_EINVAL, "negative row range");
    if (num_rows > 0 && (!out_atoms || !out_coefs)) return fail(SCOUP_EINVAL, "NULL output");
    if (!W_rows && first_row + num_rows > h->Npad) return fail(SCOUP_EINVAL, "row range beyond rows_padded");
    try {
        DeviceGuard dg(h->device);
        if (num_rows > 0) {
            const float* Wsrc = W_rows ? W_rows : h->W + first_row * (int64_t)h->L;
            const int64_t valid = std::max<int64_t>(0, std::min<int64_t>(num_rows, h->G - first_row));
            const bool dev_out = is_device_ptr(out_atoms) && is_device_ptr(out_coefs);
            uint32_t* da = out_atoms;
            float* dc = out_coefs;
            if (!dev_out) {
                dalloc(&da, (size_t)num_rows * h->K, h->stream);
                dalloc(&dc, (size_t)num_rows * h->K, h->stream);
            }
            if (h->timing) {
                if (!h->topk_ev[0]) {
                    CK(cudaEventCreate(&h->topk_ev[0]));
                    CK(cudaEventCreate(&h->topk_ev[1]));
                }
                CK(cudaEventRecord(h->topk_ev[0], h->stream));
            }
            launch_topk(Wsrc, num_rows, valid, h->L, h->K, da, dc, h->stream);
            h->kernel_launches += 1;
            if (h->timing) {
                CK(cudaEventRecord(h->topk_ev[1], h->stream));
                CK(cudaEventSynchronize(h->topk_ev[1]));
                float ms = 0;
                CK(cudaEventElapsedTime(&ms, h->topk_ev[0], h->topk_ev[1]));
                h->t_topk += ms;
            }
            CK(cudaGetLastError());
            if (!dev_out) {
                CK(cudaMemcpyAsync(out_atoms, da, sizeof(uint32_t) * num_rows * h->K, cudaMemcpyDeviceToHost, h->stream));
                CK(cudaMemcpyAsync(out_coefs, dc, sizeof(float) * num_rows * h->K, cudaMemcpyDeviceToHost, h->stream));
                dfree(da, h->stream);
                dfree(dc, h->stream);
            }
        }
        CK(cudaStreamSynchronize(h->stream));
        return check_latched(h);
    } catch (const CudaError& e) {
        return fail(SCOUP_ECUDA, std::string("CUDA error in ") + e.where + ": " + cudaGetErrorString(e.err));
    }
}

scoup_status scoup_uplift_reset(scoup_uplift* h) {
    g_last_error.clear();
    if (!h) return fail(SCOUP_EINVAL, "handle is NULL");
    try {
        DeviceGuard dg(h->device);
        CK(cudaMemsetAsync(h->W, 0, sizeof(float) * std::max<int64_t>(1, h->Npad) * h->L, h->stream));
        CK(cudaMemsetAsync(h->Z, 0, sizeof(float) * std::max<int64_t>(1, h->Npad), h->stream));
        CK(cudaMemsetAsync(h->d_stats, 0, 5 * sizeof(unsigned long long), h->stream));
        CK(cudaMemsetAsync(h->d_err_code, 0, sizeof(int), h->stream));
        h->latched = false;
        h->host_entries = 0;
        h->kernel_launches = 0;
        h->cub_launches = 0;
    } catch (const CudaError& e) {
        return fail(SCOUP_ECUDA, std::string("CUDA error in ") + e.where + ": " + cudaGetErrorString(e.err));
    }
    return SCOUP_OK;
}

scoup_status scoup_uplift_get_accumulators(scoup_uplift* h, float** W, float** Z, int64_t* rows_padded) {
    if (!h) return fail(SCOUP_EINVAL, "handle is NULL");
    if (W) *W = h->W;
    if (Z) *Z = h->Z;
    if (rows_padded) *rows_padded = h->Npad;
    return SCOUP_OK;
}

scoup_status scoup_uplift_get_stats(scoup_uplift* h, scoup_stats* out) {
    g_last_error.clear();
    if (!h || !out) return fail(SCOUP_EINVAL, "NULL argument");
    try {
        DeviceGuard dg(h->device);
        unsigned long long s[5];
        CK(cudaStreamSynchronize(h->stream));
        CK(cudaMemcpy(s, h->d_stats, sizeof(s), cudaMemcpyDeviceToHost));
        out->views = (int64_t)s[0];
        out->contributions = (int64_t)s[1];
        out->tile_entries = h->host_entries;
        out->visible = (int64_t)s[3];
        out->support_tests = (int64_t)s[4];
        out->kernel_launches = h->kernel_launches;
        out->cub_launches = h->cub_launches;
        return check_latched(h);
    } catch (const CudaError& e) {
        return fail(SCOUP_ECUDA, std::string("CUDA error in ") + e.where + ": " + cudaGetErrorString(e.err));
    }
}

scoup_status scoup_uplift_set_timing(scoup_uplift* h, int enable) {
    g_last_error.clear();
    if (!h) return fail(SCOUP_EINVAL, "handle is NULL");
    try {
        DeviceGuard dg(h->device);
        for (int i = 0; i < 2; i++)
            for (auto& es : h->ctx[i].evs) ev_accumulate(h, es);
        h->timing = enable != 0;
        h->t_pre = h->t_bin = h->t_ras = h->t_topk = 0;
        h->ras_launches = h->views_timed = 0;
    } catch (const CudaError& e) {
        return fail(SCOUP_ECUDA, std::string("CUDA error in ") + e.where + ": " + cudaGetErrorString(e.err));
    }
    return SCOUP_OK;
}

scoup_status scoup_uplift_get_timing(scoup_uplift* h, scoup_timing* out) {
    g_last_error.clear();
    if (!h || !out) return fail(SCOUP_EINVAL, "NULL argument");
    try {
        DeviceGuard dg(h->device);
        for (int i = 0; i < 2; i++)
            for (auto& es : h->ctx[i].evs) ev_accumulate(h, es);
        out->preprocess_ms = h->t_pre;
        out->binning_ms = h->t_bin;
        out->raster_ms = h->t_ras;
        out->topk_ms = h->t_topk;
        out->raster_launches = h->ras_launches;
        out->views_timed = h->views_timed;
    } catch (const CudaError& e) {
        return fail(SCOUP_ECUDA, std::string("CUDA error in ") + e.where + ": " + cudaGetErrorString(e.err));
    }
    return SCOUP_OK;
}

void scoup_uplift_free(scoup_uplift* h) {
    if (!h) return;
    DeviceGuard dg(h->device);
    if (h->stream) cudaStreamSynchronize(h->stream);
    for (int i = 0; i < 2; i++) {
        if (h->ctx[i].s) cudaStreamSynchronize(h->ctx[i].s);
        ctx_free(h->ctx[i], h->stream);
        if (h->ev_join[i]) cudaEventDestroy(h->ev_join[i]);
    }
    if (h->ev_fork) cudaEventDestroy(h->ev_fork);
    for (int i = 0; i < 2; i++)
        if (h->topk_ev[i]) cudaEventDestroy(h->topk_ev[i]);
    void* ptrs[] = {h->pg.a, h->pg.b, h->pg.c, h->d_err_code, h->d_err_index, h->d_stats, h->code_atoms,
                    h->code_coefs, h->code_atoms_in, h->code_coefs_in};
    for (void* p : ptrs) dfree(p, h->stream);
    if (h->own_wz) {
        dfree(h->W, h->stream);
        dfree(h->Z, h->stream);
    }
    cudaStreamSynchronize(h->stream);
    delete h;
}

}  // extern "C"
