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
#include <cublas_v2.h>
#include <cuda.h>
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/iterator/transform_input_iterator.cuh>

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
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

// One pipeline context: the buffers of one view batch, the stream it runs on, and where the
// batch is in its sequence of steps (DESIGN.md §5 a3).  Two contexts alternate, so that while
// the host waits for one context's counts, the GPU runs the other context's queued work.
enum Step : int { ST_IDLE = 0, ST_NEAR_FRONT, ST_NEAR_CHUNK, ST_NEAR_RASTER, ST_FAR_FRONT, ST_FAR_RASTER };

struct Ctx {
    cudaStream_t s = nullptr;     // the batch's steps (high priority: the front's short kernels)
    cudaStream_t rs = nullptr;    // its raster launches (low priority), joined back into s
    cudaEvent_t ev = nullptr;     // end of the last enqueued step (the host waits on it)
    cudaEvent_t ev_rs0 = nullptr, ev_rs1 = nullptr;  // s -> rs -> s hand-offs around a raster
    int map_ch0 = 0, map_ch1 = -1;  // host-map copy chunks the batch's rasters wait for (none: ch1 < ch0)
    ViewBuffers vb{};
    size_t g_cap = 0, s_cap = 0, e_cap = 0, t_cap = 0, px_cap = 0, tl_cap = 0, bc_cap = 0, eb_cap = 0, ee_cap = 0;
    void* cub_tmp = nullptr;
    size_t cub_cap = 0;
    // pinned host staging
    uint32_t* h_hist = nullptr;   // [MAX_VB * NHIST]
    uint32_t* h_thr = nullptr;    // [MAX_VB]
    uint64_t* h_total = nullptr;  // entries of the chunk
    int* h_nsel = nullptr;        // selected elements of the far chunk
    CamBatch* h_cams = nullptr;
    // the batch in flight
    Step step = ST_IDLE;
    int v0 = 0, nv = 0;
    int key_bits = 31;
    Binning bn{};          // the batch's bins (the adaptive bin size may change between batches)
    int64_t nsel = 0;
    bool far_any = false;
    CamBatch cams{};
    const uint32_t* ids_dev[MAX_VB][MAX_LEV] = {};
    int64_t far_cand = 0;  // visible Gaussians beyond the near split (for the near-fraction feedback)
    // timing: ring of event sets, 7 marks per batch (see ev_accumulate)
    struct EvSet { cudaEvent_t e[7]; bool pending; int views; };
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
    int nlev = 1;  // semantic levels fused per pass; W is [nlev][Npad][L]
    float* W = nullptr;
    float* Z = nullptr;
    bool own_wz = false;
    PackedGaussians pg{};
    int* d_err_code = nullptr;
    long long* d_err_index = nullptr;
    unsigned long long* d_stats = nullptr;  // views, contributions, global reds, visible, support tests, lane evaluations
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
    // near chunk: this fraction of each view's visible Gaussians.  Adapted between batches unless
    // fixed by SCOUP_NEAR_FRAC: when most Gaussians beyond the split still reach a live tile (a
    // compact scene), the split prunes little and the fraction doubles (<= 0.5); when almost
    // none do (a deep scene whose tiles saturate early), it halves back (>= 0.05).  Any split is
    // exact (DESIGN.md §5 a3), so this only moves work between the two chunks.
    double near_frac = 0.05;
    bool near_frac_fixed = false;
    int bin_shift = 0;                  // bins of 2^bin_shift px squares fixed by SCOUP_BIN_SHIFT (0: adaptive)
    int bin_shift_auto = 0;             // adaptive bin size (0: not yet chosen for this image width)
    int bin_width = 0;                  // image width the adaptive choice was made for
    int64_t bin_changes = 0;
    bool count_tests = false;           // instrumented raster: contributions + support tests (set_counters)
    int nctx = 2;                       // pipeline contexts in use (set_pipeline)
    int raster_kernel = 2;              // 2: two-pixel kernel where supported; 1: raster.cu (SCOUP_RASTER=1, A/B)
    int64_t batches[2] = {0, 0};        // view batches per context (stats)
    int64_t near_frac_changes = 0;      // in-call adaptations of near_frac (stats)
    int64_t host_map_chunks = 0;        // up-front region-map copy chunks (stats)
    cublasHandle_t blas = nullptr;      // decode GEMM (Eq. 8), created on first use
    // host region maps: the whole call's maps are copied up front on a copy stream, in chunks of
    // MAX_VB views with one event each, so the PCIe transfer runs ahead of the batches
    cudaStream_t copy_s = nullptr;
    std::vector<cudaEvent_t> chunk_ev;
    uint32_t* ids_all = nullptr;
    size_t ids_all_cap = 0;
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
    if (code == ERR_REGION) {
        const long long level = idx >> 48, pix = idx & ((1LL << 48) - 1);
        return fail(SCOUP_EDATA, "data error: region id >= num_regions at flat pixel index " + std::to_string(pix) +
                                     " (level " + std::to_string(level) + ")");
    }
    const char* what = code == ERR_GAUSSIAN ? "non-finite or invalid Gaussian parameters at Gaussian index "
                                            : "invalid code slot (atom >= L or bad coefficient) at flat slot index ";
    return fail(SCOUP_EDATA, std::string("data error: ") + what + std::to_string(idx));
}

void ctx_init(Ctx& c) {
    // stream priorities: while one context's raster fills the GPU, the other context's front
    // kernels (depth pass, selections, sorts, emission) are scheduled ahead of the raster's
    // pending CTAs as SMs free up, so the front runs in the raster's shadow
    int least = 0, greatest = 0;
    CK(cudaDeviceGetStreamPriorityRange(&least, &greatest));
    CK(cudaStreamCreateWithPriority(&c.s, cudaStreamNonBlocking, greatest));
    CK(cudaStreamCreateWithPriority(&c.rs, cudaStreamNonBlocking, least));
    CK(cudaEventCreateWithFlags(&c.ev, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&c.ev_rs0, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&c.ev_rs1, cudaEventDisableTiming));
    CK(cudaMallocHost((void**)&c.h_hist, sizeof(uint32_t) * MAX_VB * NHIST));
    CK(cudaMallocHost((void**)&c.h_thr, sizeof(uint32_t) * MAX_VB));
    CK(cudaMallocHost((void**)&c.h_total, sizeof(uint64_t)));
    CK(cudaMallocHost((void**)&c.h_nsel, sizeof(int)));
    CK(cudaMallocHost((void**)&c.h_cams, sizeof(CamBatch)));
}

void ctx_free(Ctx& c, cudaStream_t s) {
    for (auto& es : c.evs)
        for (int k = 0; k < 7; k++) cudaEventDestroy(es.e[k]);
    c.evs.clear();
    ViewBuffers& b = c.vb;
    void* ptrs[] = {b.code, b.hist, b.thr, b.cams, b.sel, b.nsel, b.skey, b.skey_alt, b.sval, b.sval_sorted,
                    b.tiles, b.rect, b.rec0, b.rec1, b.rec2, b.rec3, b.trect, b.selcnt, b.live_sat, b.Tstate,
                    b.tile_live, b.eval, b.ranges, b.bcnt, b.ebin, b.eel, b.binfo, c.cub_tmp};
    for (void* p : ptrs) dfree(p, s);
    void* hp[] = {c.h_hist, c.h_thr, c.h_total, c.h_nsel, c.h_cams};
    for (void* p : hp)
        if (p) cudaFreeHost(p);
    if (c.ev) cudaEventDestroy(c.ev);
    if (c.ev_rs0) cudaEventDestroy(c.ev_rs0);
    if (c.ev_rs1) cudaEventDestroy(c.ev_rs1);
    if (c.rs) {
        cudaStreamSynchronize(c.rs);
        cudaStreamDestroy(c.rs);
    }
    if (c.s) cudaStreamDestroy(c.s);
    c = Ctx{};
}

void ctx_reserve_cub(Ctx& c, size_t bytes) { grow((char**)&c.cub_tmp, &c.cub_cap, bytes, c.s); }

// Per-selected-element buffers (EWA records, sort keys, bin counts) for a chunk of n elements:
// grown on demand (stream-ordered on the context's stream, after every earlier reader).
void ctx_reserve_sel(Ctx& c, int64_t n) {
    ViewBuffers& b = c.vb;
    n = std::max<int64_t>(n, 1);
    if ((size_t)n <= c.s_cap && b.rec0) return;
    const size_t cap = (size_t)((double)n * 1.25);
    void* ptrs[] = {b.skey, b.skey_alt, b.sval, b.sval_sorted, b.tiles, b.rect,
                    b.rec0, b.rec1, b.rec2, b.rec3};
    for (void* p : ptrs) dfree(p, c.s);
#define RG(f) { dalloc(&b.f, cap, c.s); }
    RG(skey) RG(skey_alt) RG(sval) RG(sval_sorted) RG(tiles) RG(rect) RG(rec0) RG(rec1) RG(rec2) RG(rec3)
#undef RG
    c.s_cap = cap;
}

// Per-(view, Gaussian) buffers for batches of up to B*G elements, per-pixel state for
// B views of npx pixels, tile flags for B*ntiles tiles.
void ctx_reserve(Ctx& c, int64_t G, int B, int64_t pixels, int64_t tiles) {
    ViewBuffers& b = c.vb;
    const int64_t n = std::max<int64_t>((int64_t)B * G, 1);
    if ((size_t)n > c.g_cap || !b.code) {
        void* ptrs[] = {b.code, b.sel, b.trect, b.selcnt};
        for (void* p : ptrs) dfree(p, c.s);
#define RG(f) { dalloc(&b.f, (size_t)n, c.s); }
        RG(sel) RG(trect)
#undef RG
        dalloc(&b.code, (size_t)n + 4, c.s);  // (preprocess reads the aligned 16 B holding a code)
        dalloc(&b.selcnt, select_counts_needed(G, MAX_VB) + 1, c.s);
        c.g_cap = (size_t)n;
    }
    if (!b.hist) {
        dalloc(&b.hist, (size_t)MAX_VB * NHIST, c.s);
        dalloc(&b.thr, MAX_VB, c.s);
        dalloc(&b.cams, 1, c.s);
        dalloc(&b.nsel, 1, c.s);
    }
    grow(&b.Tstate, &c.px_cap, (size_t)std::max<int64_t>(pixels, 1), c.s, 1.0);
    if ((size_t)std::max<int64_t>(tiles, 1) > c.tl_cap || !b.tile_live) {
        dfree(b.live_sat, c.s);
        dalloc(&b.live_sat, (size_t)MAX_VB * MAX_SAT_ENTRIES, c.s);
    }
    grow(&b.tile_live, &c.tl_cap, (size_t)std::max<int64_t>(tiles, 1), c.s, 1.0);
}

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


constexpr int EV_RING = 8;

// Marks per batch: 0 start, 1 near front done, 2 near raster start, 3 near raster end,
// 4 far front done, 5 far raster start, 6 far raster end.
void ev_accumulate(scoup_uplift* h, Ctx::EvSet& es) {
    if (!es.pending) return;
    CK(cudaEventSynchronize(es.e[6]));
    float t[6];
    for (int k = 0; k < 6; k++) CK(cudaEventElapsedTime(&t[k], es.e[k], es.e[k + 1]));
    h->t_pre += t[0] + t[3];
    h->t_bin += t[1] + t[4];
    h->t_ras += t[2] + t[5];
    h->ras_launches++;
    h->views_timed += es.views;
    es.pending = false;
}

Ctx::EvSet* ev_begin(scoup_uplift* h, Ctx& c) {
    if (!h->timing) { c.ev_cur = -1; return nullptr; }
    if (c.evs.empty()) {
        c.evs.resize(EV_RING);
        for (auto& es : c.evs) {
            for (int k = 0; k < 7; k++) CK(cudaEventCreate(&es.e[k]));
            es.pending = false;
        }
    }
    c.ev_cur = c.ev_next;
    c.ev_next = (c.ev_next + 1) % EV_RING;
    Ctx::EvSet& es = c.evs[c.ev_cur];
    ev_accumulate(h, es);
    return &es;
}

void ev_mark(Ctx& c, int k, cudaStream_t st = nullptr) {
    if (c.ev_cur >= 0) CK(cudaEventRecord(c.evs[c.ev_cur].e[k], st ? st : c.s));
}

// Bins: squares of 2^bin_shift px (default 64x64, SCOUP_BIN_SHIFT) holding the depth-ordered
// candidates of the 16x16 tiles inside them; each tile filters its bin's list (band_relevant).
Binning choose_binning(int Wd, int Hd, int bin_shift) {
    // default: 64 px bins for wide images, 32 px below 1280 px (measured: outdoor 1600 px, indoor
    // 988 px and small 512 px configs); SCOUP_BIN_SHIFT fixes it
    if (bin_shift <= 0) bin_shift = Wd >= 1280 ? 6 : 5;
    Binning b;
    b.tiles_x = (Wd + TILE - 1) / TILE;
    b.tiles_y = (Hd + TILE - 1) / TILE;
    b.bshx = b.bshy = bin_shift;
    b.bins_x = (Wd + (1 << bin_shift) - 1) >> bin_shift;
    b.bins_y = (Hd + (1 << bin_shift) - 1) >> bin_shift;
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

// Per-call context of add_views shared by the steps.
struct CallArgs {
    const Camera* cams;
    Binning bn;
    const int64_t* code_row0;    // [nlev][V]: first row of (level, view) in the combined code table
    const int32_t* num_regions;  // [nlev][V]
    int V;
    int S;
    long long* contrib_out;
    int64_t npx;
    bool dense;
    // render (Eq. 7) instead of uplift
    bool render = false;
    const uint32_t* r_atoms = nullptr;
    const float* r_coefs = nullptr;
    int rK = 0;
    float* r_out = nullptr;
};

// Split histogram of a batch (sampled depth codes, per view -> host), camera copy for the passes.
void step_depth(scoup_uplift* h, Ctx& c, const CallArgs& a) {
    ViewBuffers& b = c.vb;
    Ctx::EvSet* es = ev_begin(h, c);
    if (es) es->views = c.nv;
    ev_mark(c, 0);
    c.cams.n = c.nv;
    for (int v = 0; v < c.nv; v++) c.cams.cam[v] = a.cams[c.v0 + v];
    *c.h_cams = c.cams;
    CK(cudaMemcpyAsync(b.cams, c.h_cams, sizeof(CamBatch), cudaMemcpyHostToDevice, c.s));
    CK(cudaMemsetAsync(b.hist, 0, sizeof(uint32_t) * NHIST * c.nv, c.s));
    launch_depth_hist(h->pg, h->G, c.cams, c.key_bits, b.hist, c.s);
    CK(cudaMemcpyAsync(c.h_hist, b.hist, sizeof(uint32_t) * NHIST * c.nv, cudaMemcpyDeviceToHost, c.s));
    CK(cudaEventRecord(c.ev, c.s));
    h->kernel_launches += 1;
    c.step = ST_NEAR_FRONT;
}

// Front of one chunk on the nsel selected elements: EWA preprocess, depth sort, per-segment bin
// counts of the bin scatter (binsort.cu), entry total -> host.
void chunk_front(scoup_uplift* h, Ctx& c, const CallArgs& a, int64_t nsel) {
    (void)a;
    ViewBuffers& b = c.vb;
    c.nsel = nsel;
    if (nsel <= 0) return;
    ctx_reserve_sel(c, nsel);
    int vbits = 0;
    while ((1 << vbits) < c.nv) vbits++;
    const int end_bit = c.key_bits + vbits;
    launch_preprocess(h->pg, h->G, c.cams, c.bn, b, c.key_bits, nsel, c.s);
    size_t need = 0;
    CK(cub::DeviceRadixSort::SortPairs(nullptr, need, b.skey, b.skey_alt, b.sval, b.sval_sorted, (int)nsel, 0, end_bit,
                                       c.s));
    ctx_reserve_cub(c, need);
    CK(cub::DeviceRadixSort::SortPairs(c.cub_tmp, need, b.skey, b.skey_alt, b.sval, b.sval_sorted, (int)nsel, 0,
                                       end_bit, c.s));
    // entry counts in sorted order, scanned in place into b.skey (dead after the sort): the
    // binning's entry offsets; the exact total -> host
    if (!b.binfo) dalloc(&b.binfo, 1, c.s);
    launch_binsort_gather(b.sval_sorted, b.tiles, nsel, b.skey, b.binfo, c.s);
    size_t need2 = 0;
    CK(cub::DeviceScan::InclusiveSum(nullptr, need2, b.skey, b.skey, (int)nsel, c.s));
    ctx_reserve_cub(c, need2);
    CK(cub::DeviceScan::InclusiveSum(c.cub_tmp, need2, b.skey, b.skey, (int)nsel, c.s));
    CK(cudaMemcpyAsync(c.h_total, &b.binfo->total, sizeof(uint64_t), cudaMemcpyDeviceToHost, c.s));
    h->kernel_launches += 2;
    // CUB kernels: the onesweep sort (histogram, exclusive sum, one pass per 8 key bits) and the
    // scan (init + scan)
    h->cub_launches += 2 + (end_bit + 7) / 8 + 2;
}

// Near chunk: per view, the nearest ~near_frac of the visible Gaussians (a histogram bucket
// boundary of the depth code), stable-compacted, then the chunk front.
void step_near_front(scoup_uplift* h, Ctx& c, const CallArgs& a) {
    CK(cudaEventSynchronize(c.ev));
    const uint32_t none = (1u << c.key_bits) - 1u;
    const int shift = c.key_bits > HIST_BITS ? c.key_bits - HIST_BITS : 0;
    c.far_any = false;
    c.far_cand = 0;
    for (int v = 0; v < c.nv; v++) {
        // the histogram samples every HIST_SAMPLE-th Gaussian: the split follows the sample's
        // quantile; the exact near count comes back from the compaction (next step)
        const uint32_t* hv = c.h_hist + (int64_t)v * NHIST;
        uint64_t total = 0;
        for (int k = 0; k < NHIST; k++) total += hv[k];
        const uint64_t target = (uint64_t)std::ceil(h->near_frac * (double)total);
        uint32_t thr = none;  // everything visible
        uint64_t cum = total;
        if (target < total) {
            cum = 0;
            for (int k = 0; k < NHIST; k++) {
                cum += hv[k];
                if (cum >= target) {
                    thr = (uint32_t)std::min<uint64_t>((uint64_t)(k + 1) << shift, none);
                    break;
                }
            }
        }
        if (thr != none) c.far_any = true;  // (unsampled Gaussians may lie beyond the split)
        c.h_thr[v] = thr;
        c.far_cand += (int64_t)(total - cum) * HIST_SAMPLE;
    }
    ViewBuffers& b = c.vb;
    CK(cudaMemcpyAsync(b.thr, c.h_thr, sizeof(uint32_t) * c.nv, cudaMemcpyHostToDevice, c.s));
    // the full depth pass: codes, reach boxes and the near chunk's compaction in one sweep
    launch_depth_pass_near(h->pg, h->G, c.cams, c.key_bits, b.thr, b.code, h->d_stats + 3, latch_of(h), a.bn, b.trect,
                           b.selcnt, b.sel, b.nsel, c.s);
    h->kernel_launches += 3;
    CK(cudaMemcpyAsync(c.h_nsel, b.nsel, sizeof(int), cudaMemcpyDeviceToHost, c.s));
    CK(cudaEventRecord(c.ev, c.s));
    c.step = ST_NEAR_CHUNK;
}

// Near chunk front on the exact number of selected elements.
void step_near_chunk(scoup_uplift* h, Ctx& c, const CallArgs& a) {
    CK(cudaEventSynchronize(c.ev));
    chunk_front(h, c, a, (int64_t)*c.h_nsel);
    ev_mark(c, 1);
    CK(cudaEventRecord(c.ev, c.s));
    c.step = ST_NEAR_RASTER;
}

// Back of one chunk: emit (tile-exact), tile sort, ranges, raster.  Chunk 0 always launches the
// raster so that every tile initialises its transmittance state.
scoup_status chunk_back(scoup_uplift* h, Ctx& c, const CallArgs& a, int chunk, int mark0) {
    ViewBuffers& b = c.vb;
    const uint64_t E = c.nsel > 0 ? *c.h_total : 0;
    const int ntiles = c.bn.nbins() * c.nv;  // bins of the batch (= the ranges' sentinel key)
    if (E >= (uint64_t)INT32_MAX)
        return fail(SCOUP_EUNSUPPORTED, "view batch produces " + std::to_string(E) + " tile entries (>= 2^31)");
    if ((size_t)ntiles > c.t_cap || !b.ranges) {
        dfree(b.ranges, c.s);
        dalloc(&b.ranges, ntiles, c.s);
        c.t_cap = ntiles;
    }
    h->host_entries += (int64_t)E;
    if (chunk == 0 && h->bin_shift == 0 && c.nsel > 0) {
        // adaptive bin size for later batches: bins covered per near-chunk element.  Large
        // footprints (many bins each) make the entry sort dominate -> larger bins; small ones
        // make every tile filter a long list of Gaussians that miss it -> smaller bins
        // (measured: configs[4] 1570 -> 1145 ms with 128-px instead of 64-px bins; outdoor and
        // indoor stay at their width-based defaults)
        const double per = (double)E / (double)c.nsel;
        const int cur = c.bn.bshx;
        int nxt = cur;
        if (per > 12.0 && cur < 8) nxt = cur + 1;
        else if (per < 1.5 && cur > 5) nxt = cur - 1;
        if (nxt != cur && nxt != h->bin_shift_auto) {
            h->bin_shift_auto = nxt;
            h->bin_changes++;
        }
    }
    if (E == 0 && chunk > 0) {
        ev_mark(c, mark0);
        ev_mark(c, mark0 + 1);
        return SCOUP_OK;
    }
    if (E > 0) {
        grow(&b.eval, &c.e_cap, (size_t)E, c.s);
        const int nb = c.bn.nbins();
        const size_t nseg = binsort_segments_max((int64_t)E, c.nv);
        grow(&b.bcnt, &c.bc_cap, nseg * (size_t)nb, c.s);
        grow(&b.ebin, &c.eb_cap, (size_t)E, c.s);
        grow(&b.eel, &c.ee_cap, (size_t)E, c.s);
        launch_binsort(b.selcnt, select_tiles_per_view(h->G), b.skey, b.sval_sorted, b.rect, c.nsel, (int64_t)E, c.nv,
                       c.bn.bins_x, nb, b.binfo, b.bcnt, b.ebin, b.eel, b.ranges, b.eval, c.s);
        h->kernel_launches += 5;
    } else {
        CK(cudaMemsetAsync(b.ranges, 0, sizeof(uint2) * ntiles, c.s));
    }
    RasterParams p{};
    p.nviews = c.nv;
    p.width = a.cams[c.v0].width;
    p.height = a.cams[c.v0].height;
    p.G = h->G;
    p.bn = c.bn;
    p.ranges = b.ranges;
    p.eval = b.eval;
    p.rec0 = b.rec0;
    p.rec1 = b.rec1;
    p.rec2 = b.rec2;
    p.rec3 = b.rec3;
    p.Tstate = b.Tstate;
    p.tile_live = b.tile_live;
    p.chunk = chunk;
    p.count_tests = h->count_tests || a.contrib_out != nullptr;
    p.dense = a.dense;
    p.r_atoms = a.r_atoms;
    p.r_coefs = a.r_coefs;
    p.rK = a.rK;
    p.r_out = a.r_out;
    p.r_view0 = c.v0;
    p.nlev = h->nlev;
    for (int v = 0; v < c.nv; v++) {
        const int u = c.v0 + v;
        for (int l = 0; l < (a.render ? 0 : h->nlev); l++) {  // the render reads no region maps
            p.region_ids[v][l] = c.ids_dev[v][l];
            p.code_row0[v][l] = a.code_row0[(int64_t)l * a.V + u];
            p.num_regions[v][l] = a.num_regions[(int64_t)l * a.V + u];
        }
        p.pixel_base[v] = (long long)u * a.npx;
        p.contrib_out[v] = a.contrib_out ? a.contrib_out + u : nullptr;
    }
    p.code_atoms = h->code_atoms;
    p.code_coefs = h->code_coefs;
    p.S = a.S;
    p.L = h->L;
    p.W = h->W;
    p.W_level_stride = h->Npad * (int64_t)h->L;
    p.Z = h->Z;
    p.contrib_ctr = h->d_stats + 1;
    p.support_ctr = h->d_stats + 4;
    p.lane_eval_ctr = h->d_stats + 5;
    p.red_ctr = h->d_stats + 2;
    p.err = latch_of(h);
    // the raster on the context's low-priority stream, joined back before the next step
    CK(cudaEventRecord(c.ev_rs0, c.s));
    CK(cudaStreamWaitEvent(c.rs, c.ev_rs0, 0));
    // only the raster reads the region maps: the batch's front runs while its chunk is still in flight
    for (int j = c.map_ch0; j <= c.map_ch1; j++) CK(cudaStreamWaitEvent(c.rs, h->chunk_ev[j], 0));
    ev_mark(c, mark0, c.rs);
    if (a.render) launch_render(p, c.rs);
    else if (h->raster_kernel != 1 && raster2_supported(p)) launch_raster2(p, c.rs);
    else launch_raster(p, c.rs);
    ev_mark(c, mark0 + 1, c.rs);
    CK(cudaEventRecord(c.ev_rs1, c.rs));
    CK(cudaStreamWaitEvent(c.s, c.ev_rs1, 0));
    h->kernel_launches += 1;
    return SCOUP_OK;
}

// Near raster, then the far selection: visible Gaussians beyond the split whose conservative
// reach touches a tile that is still live (count -> host).
scoup_status step_near_raster(scoup_uplift* h, Ctx& c, const CallArgs& a) {
    CK(cudaEventSynchronize(c.ev));
    scoup_status st = chunk_back(h, c, a, 0, 2);
    if (st != SCOUP_OK) return st;
    if (c.far_any) {
        launch_select_far2(c.vb, h->pg, h->G, c.nv, c.key_bits, c.bn, c.vb.selcnt, c.s);
        h->kernel_launches += 4;
        CK(cudaMemcpyAsync(c.h_nsel, c.vb.nsel, sizeof(int), cudaMemcpyDeviceToHost, c.s));
    }
    CK(cudaEventRecord(c.ev, c.s));
    c.step = ST_FAR_FRONT;
    return SCOUP_OK;
}

void step_far_front(scoup_uplift* h, Ctx& c, const CallArgs& a) {
    CK(cudaEventSynchronize(c.ev));
    if (!h->near_frac_fixed && c.far_any && c.far_cand > 0) {
        const double kept = (double)*c.h_nsel / (double)c.far_cand;
        const double before = h->near_frac;
        if (kept > 0.25) h->near_frac = std::min(0.5, h->near_frac * 2.0);
        else if (kept < 0.05) h->near_frac = std::max(0.05, h->near_frac * 0.5);
        if (h->near_frac != before) h->near_frac_changes++;
    }
    chunk_front(h, c, a, c.far_any ? (int64_t)*c.h_nsel : 0);
    ev_mark(c, 4);
    CK(cudaEventRecord(c.ev, c.s));
    c.step = ST_FAR_RASTER;
}

scoup_status step_far_raster(scoup_uplift* h, Ctx& c, const CallArgs& a) {
    CK(cudaEventSynchronize(c.ev));
    scoup_status st = chunk_back(h, c, a, 1, 5);
    if (c.ev_cur >= 0) c.evs[c.ev_cur].pending = true;
    c.step = ST_IDLE;
    return st;
}

__global__ void add_u64(unsigned long long* p, unsigned long long v) { atomicAdd(p, v); }

// The per-view pipeline shared by the uplift and the render: view batches through the two
// contexts' step machines (depth pass, near chunk, near raster + far selection, far chunk, far
// raster), joined back into the handle's stream.  region_ids: nlev per-level maps (uplift) or
// none (render).
scoup_status run_views(scoup_uplift* h, int32_t num_views, const scoup_camera* cameras, const Binning& bn,
                       int64_t npx, CallArgs& args, const uint32_t* const* region_ids, int nlev) {
    try {
        bool ids_on_device = true;
        for (int l = 0; l < nlev; l++) ids_on_device = ids_on_device && is_device_ptr(region_ids[l]);
        std::vector<Camera> cams(num_views);
        for (int v = 0; v < num_views; v++) cams[v] = to_cam(cameras[v]);
        // ---- view batches: up to MAX_VB views per pass (bounded by the bin table and by the
        // depth-code width: view bits + code bits <= 32)
        const int Bmax = std::max(1, std::min(MAX_VB, (int)num_views));
        const int ntiles = bn.tiles_x * bn.tiles_y;
        // ---- fork the two pipeline contexts off the caller's stream
        CK(cudaEventRecord(h->ev_fork, h->stream));
        for (int i = 0; i < 2; i++) {
            CK(cudaStreamWaitEvent(h->ctx[i].s, h->ev_fork, 0));
            ctx_reserve(h->ctx[i], h->G, Bmax, (int64_t)Bmax * npx, (int64_t)Bmax * ntiles);
        }
        args.cams = cams.data();
        if (!ids_on_device && nlev > 0) {
            // all views' maps (every level) to the device on the copy stream, chunk by chunk
            if (!h->copy_s) CK(cudaStreamCreateWithFlags(&h->copy_s, cudaStreamNonBlocking));
            const int nch = (num_views + MAX_VB - 1) / MAX_VB;
            while ((int)h->chunk_ev.size() < nch) {
                cudaEvent_t e = nullptr;
                CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
                h->chunk_ev.push_back(e);
            }
            grow(&h->ids_all, &h->ids_all_cap, (size_t)nlev * num_views * npx, h->stream, 1.0);
            CK(cudaEventRecord(h->ev_fork, h->stream));  // the buffer (and earlier readers) are done
            CK(cudaStreamWaitEvent(h->copy_s, h->ev_fork, 0));
        }
        // Host maps: chunk j (MAX_VB views, every level) is enqueued on the copy stream a few
        // chunks ahead of the batches that read it.  (Enqueueing the whole call's 2 GB at once
        // blocked the host thread in cudaMemcpyAsync until most of it had been copied -- the
        // copy queue is bounded -- so the first batches started only after the transfer:
        // measured +37 ms on the outdoor step, the whole PCIe time.)
        const int nch_all = (!ids_on_device && nlev > 0) ? (num_views + MAX_VB - 1) / MAX_VB : 0;
        int copied = 0;  // chunks enqueued
        auto copy_ahead = [&](int upto) {
            for (; copied < std::min(upto, nch_all); copied++) {
                const int v0 = copied * MAX_VB, nv = std::min(MAX_VB, num_views - v0);
                for (int l = 0; l < nlev; l++)
                    CK(cudaMemcpyAsync(h->ids_all + ((int64_t)l * num_views + v0) * npx,
                                       region_ids[l] + (int64_t)v0 * npx, sizeof(uint32_t) * npx * nv,
                                       cudaMemcpyHostToDevice, h->copy_s));
                CK(cudaEventRecord(h->chunk_ev[copied], h->copy_s));
                h->host_map_chunks++;
            }
        };
        copy_ahead(3);
        int next = 0;  // first view not yet assigned to a batch
        auto start_batch = [&](Ctx& c) {
            int B = std::min(Bmax, num_views - next);
            int kb = 31;
            for (;; B = std::max(1, B / 2)) {
                int vbits = 0;
                while ((1 << vbits) < B) vbits++;
                kb = std::min(31, depth_key_bits(h, &cams[next], B));
                if (kb + vbits <= 32 || B == 1) break;
            }
            c.v0 = next;
            c.nv = B;
            c.key_bits = kb;
            next += B;
            {   // the batch's bins: fixed (SCOUP_BIN_SHIFT) or the handle's adaptive size
                const int Wd = cams[c.v0].width, Hd = cams[c.v0].height;
                if (h->bin_shift > 0) {
                    c.bn = choose_binning(Wd, Hd, h->bin_shift);
                } else {
                    if (h->bin_width != Wd) {
                        h->bin_width = Wd;
                        h->bin_shift_auto = choose_binning(Wd, Hd, 0).bshx;
                    }
                    c.bn = choose_binning(Wd, Hd, h->bin_shift_auto);
                }
            }
            if (!ids_on_device && nlev > 0) {  // this batch's chunks of the host-map copy
                copy_ahead((c.v0 + c.nv - 1) / MAX_VB + 3);
                c.map_ch0 = c.v0 / MAX_VB;
                c.map_ch1 = (c.v0 + c.nv - 1) / MAX_VB;
            } else {
                c.map_ch0 = 0;
                c.map_ch1 = -1;
            }
            for (int v = 0; v < c.nv; v++) {
                const int u = c.v0 + v;
                for (int l = 0; l < nlev; l++)
                    c.ids_dev[v][l] = ids_on_device ? region_ids[l] + (int64_t)u * npx
                                                    : h->ids_all + ((int64_t)l * num_views + u) * npx;
            }
            step_depth(h, c, args);
        };
        scoup_status st = SCOUP_OK;
        for (int ci = 0; ci < 2; ci++) h->ctx[ci].step = ST_IDLE;
        // Event-driven step machine: a context advances as soon as its last enqueued step has
        // completed (its next step needs a count read back by the host), independently of the
        // other context -- so one context can run its whole front (several short steps with host
        // round trips) while the other's raster runs.  When neither is ready, the host waits.
        auto advance = [&](int ci) {
            Ctx& c = h->ctx[ci];
            switch (c.step) {
                case ST_IDLE: start_batch(c); h->batches[ci]++; break;
                case ST_NEAR_FRONT: step_near_front(h, c, args); break;
                case ST_NEAR_CHUNK: step_near_chunk(h, c, args); break;
                case ST_NEAR_RASTER: st = step_near_raster(h, c, args); break;
                case ST_FAR_FRONT: step_far_front(h, c, args); break;
                case ST_FAR_RASTER: st = step_far_raster(h, c, args); break;
            }
        };
        for (;;) {
            bool any = false, progressed = false;
            for (int ci = 0; ci < h->nctx && st == SCOUP_OK; ci++) {
                Ctx& c = h->ctx[ci];
                if (c.step == ST_IDLE) {
                    if (next < num_views) { advance(ci); progressed = true; any = true; }
                    continue;
                }
                any = true;
                const cudaError_t q = cudaEventQuery(c.ev);
                if (q == cudaSuccess) {
                    advance(ci);
                    progressed = true;
                } else if (q != cudaErrorNotReady) {
                    CK(q);
                }
            }
            if (st != SCOUP_OK || !any) break;
            if (!progressed) std::this_thread::yield();
        }
        // ---- join back into the caller's stream
        for (int i = 0; i < 2; i++) {
            CK(cudaEventRecord(h->ev_join[i], h->ctx[i].s));
            CK(cudaStreamWaitEvent(h->stream, h->ev_join[i], 0));
        }
        if (!ids_on_device && nlev > 0) {  // (every chunk was waited on by a batch; this is the last)
            CK(cudaStreamWaitEvent(h->stream, h->chunk_ev[(num_views - 1) / MAX_VB], 0));
        }
        add_u64<<<1, 1, 0, h->stream>>>(h->d_stats + 0, (unsigned long long)num_views);
        h->kernel_launches += 1;
        CK(cudaGetLastError());
        return st;
    } catch (const CudaError& e) {
        return fail(e.err == cudaErrorMemoryAllocation ? SCOUP_ENOMEM : SCOUP_ECUDA,
                    std::string("CUDA error in ") + e.where + ": " + cudaGetErrorString(e.err));
    }
}


}  // namespace

void scoup::set_last_error(const char* msg) { g_last_error = msg ? msg : ""; }

extern "C" {

const char* scoup_last_error(void) { return g_last_error.c_str(); }

const char* scoup_version(void) { return "scoup-b200 0.1.0 (sm_100a)"; }

scoup_status scoup_uplift_init(int device, void* cuda_stream, int64_t num_gaussians, const float* means,
                               const float* scales, const float* rotations, const float* opacities, int32_t L,
                               int32_t K, float* W, float* Z, int64_t rows_padded, scoup_uplift** out) {
    return scoup_uplift_init_levels(device, cuda_stream, num_gaussians, means, scales, rotations, opacities, 1, L, K,
                                    W, Z, rows_padded, out);
}

scoup_status scoup_uplift_init_levels(int device, void* cuda_stream, int64_t num_gaussians, const float* means,
                                      const float* scales, const float* rotations, const float* opacities,
                                      int32_t num_levels, int32_t L, int32_t K, float* W, float* Z,
                                      int64_t rows_padded, scoup_uplift** out) {
    g_last_error.clear();
    if (!out) return fail(SCOUP_EINVAL, "out is NULL");
    *out = nullptr;
    if (num_gaussians < 0) return fail(SCOUP_EINVAL, "num_gaussians < 0");
    if (num_gaussians > 0 && (!means || !scales || !rotations || !opacities))
        return fail(SCOUP_EINVAL, "Gaussian parameter pointer is NULL");
    if (K < 1) return fail(SCOUP_EINVAL, "K < 1");
    if (L < 1) return fail(SCOUP_EINVAL, "L < 1");
    if (K > L) return fail(SCOUP_EINVAL, "K > L (SPEC.md:291)");
    if (num_levels < 1) return fail(SCOUP_EINVAL, "num_levels < 1");
    if (num_levels > MAX_LEV) return fail(SCOUP_EUNSUPPORTED, "num_levels > SCOUP_MAX_LEVELS");
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
        h->nlev = num_levels;
        CK(cudaDeviceGetAttribute(&h->sms, cudaDevAttrMultiProcessorCount, device));
        if (const char* e = getenv("SCOUP_CACHE_CONFIG")) {  // (A/B) device-wide L1 / shared-memory preference
            const int m = atoi(e);
            CK(cudaDeviceSetCacheConfig(m == 1 ? cudaFuncCachePreferShared : m == 2 ? cudaFuncCachePreferL1
                                                                                   : cudaFuncCachePreferNone));
        }
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
            dalloc(&h->W, (size_t)std::max<int64_t>(1, rows_padded) * L * num_levels, hs);
            dalloc(&h->Z, (size_t)std::max<int64_t>(1, rows_padded), hs);
            h->own_wz = true;
        }
        dalloc(&h->d_err_code, 1, hs);
        dalloc(&h->d_err_index, 1, hs);
        dalloc(&h->d_stats, 6, hs);
        CK(cudaMemsetAsync(h->d_err_code, 0, sizeof(int), h->stream));
        CK(cudaMemsetAsync(h->d_err_index, 0, sizeof(long long), h->stream));
        CK(cudaMemsetAsync(h->d_stats, 0, 6 * sizeof(unsigned long long), h->stream));
        CK(cudaMemsetAsync(h->W, 0, sizeof(float) * rows_padded * L * num_levels, h->stream));
        CK(cudaMemsetAsync(h->Z, 0, sizeof(float) * rows_padded, h->stream));
        const int64_t G = std::max<int64_t>(1, num_gaussians);
        dalloc(&h->pg.a, G, hs);
        dalloc(&h->pg.b, G, hs);
        dalloc(&h->pg.c, G + 1, hs);  // (preprocess reads the aligned 16 B holding c[i])
        dalloc(&h->pg.s2, G, hs);
        if (const char* nf = std::getenv("SCOUP_NEAR_FRAC")) {
            const double f = std::atof(nf);
            if (f > 0.0) {
                h->near_frac = f;
                h->near_frac_fixed = true;
            }
        }
        if (const char* rk = std::getenv("SCOUP_RASTER")) h->raster_kernel = std::atoi(rk) == 1 ? 1 : 2;
        if (const char* bs = std::getenv("SCOUP_BIN_SHIFT")) {
            const int v = std::atoi(bs);
            if (v >= 4 && v <= 10) h->bin_shift = v;
        }
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
    if (h && h->nlev != 1) return fail(SCOUP_ESTATE, "handle has several levels: use scoup_uplift_add_views_levels");
    return scoup_uplift_add_views_levels(h, num_views, cameras, &region_ids, code_row0, num_regions, &code_atoms,
                                         &code_coefs, S, contributions_out);
}

scoup_status scoup_uplift_add_views_levels(scoup_uplift* h, int32_t num_views, const scoup_camera* cameras,
                                           const uint32_t* const* region_ids, const int64_t* code_row0,
                                           const int32_t* num_regions, const uint32_t* const* code_atoms,
                                           const float* const* code_coefs, int32_t S, int64_t* contributions_out) {
    g_last_error.clear();
    if (!h) return fail(SCOUP_EINVAL, "handle is NULL");
    if (h->latched) return fail(SCOUP_ESTATE, "a latched data error is pending; call scoup_uplift_reset");
    if (num_views < 0) return fail(SCOUP_EINVAL, "num_views < 0");
    if (num_views == 0) return SCOUP_OK;
    const int nlev = h->nlev;
    if (!cameras || !region_ids || !code_row0 || !num_regions || !code_atoms || !code_coefs)
        return fail(SCOUP_EINVAL, "NULL argument");
    // code_atoms[l] == NULL for every level: dense region features (Eq. 3 baseline), S == L
    const bool dense = code_atoms[0] == nullptr;
    for (int l = 0; l < nlev; l++) {
        if (!region_ids[l] || !code_coefs[l]) return fail(SCOUP_EINVAL, "NULL level argument");
        if ((code_atoms[l] == nullptr) != dense) return fail(SCOUP_EINVAL, "code_atoms NULL for some levels only");
    }
    if (S < 1) return fail(SCOUP_EINVAL, "S < 1");
    if (dense) {
        if (S != h->L) return fail(SCOUP_EINVAL, "dense features need S == L");
    } else {
        if (S > SCOUP_MAX_S) return fail(SCOUP_EUNSUPPORTED, "S > SCOUP_MAX_S");
        if (nlev * S > SCOUP_MAX_S) return fail(SCOUP_EUNSUPPORTED, "num_levels * S > SCOUP_MAX_S");
    }
    const int Wd = cameras[0].width, Hd = cameras[0].height;
    std::vector<int64_t> rows(nlev, 0), loff(nlev, 0);
    for (int v = 0; v < num_views; v++) {
        const scoup_camera& c = cameras[v];
        if (c.width != Wd || c.height != Hd) return fail(SCOUP_EINVAL, "cameras of one call must share width/height");
        if (c.width <= 0 || c.height <= 0) return fail(SCOUP_EINVAL, "camera width/height <= 0");
        if (!(c.fx > 0.f) || !(c.fy > 0.f) || !std::isfinite(c.fx) || !std::isfinite(c.fy) || !std::isfinite(c.cx) ||
            !std::isfinite(c.cy))
            return fail(SCOUP_EINVAL, "camera " + std::to_string(v) + ": bad intrinsics");
        if (!rigid_ok(c.world_to_camera))
            return fail(SCOUP_EDATA, "camera " + std::to_string(v) + ": world_to_camera is not rigid (1e-5)");
        for (int l = 0; l < nlev; l++) {
            const int64_t k = (int64_t)l * num_views + v;
            if (code_row0[k] < 0 || num_regions[k] < 0) return fail(SCOUP_EINVAL, "negative code_row0 / num_regions");
            rows[l] = std::max<int64_t>(rows[l], code_row0[k] + num_regions[k]);
        }
    }
    if ((int64_t)Wd * Hd >= (int64_t)INT32_MAX) return fail(SCOUP_EUNSUPPORTED, "image too large");
    if ((int64_t)((Wd + TILE - 1) / TILE + 1) * ((Hd + TILE - 1) / TILE + 1) > MAX_SAT_ENTRIES)
        return fail(SCOUP_EUNSUPPORTED, "image too large for the tile tables (> 12288 16x16 tiles)");
    if (h->G == 0) return SCOUP_OK;
    const Binning bn = choose_binning(Wd, Hd, h->bin_shift);
    const int64_t npx = (int64_t)Wd * Hd;
    int64_t total_rows = 0;
    for (int l = 0; l < nlev; l++) {
        loff[l] = total_rows;
        total_rows += rows[l];
    }
    // combined code table: level l's rows start at loff[l]
    std::vector<int64_t> row0c((size_t)nlev * num_views);
    for (int l = 0; l < nlev; l++)
        for (int v = 0; v < num_views; v++)
            row0c[(size_t)l * num_views + v] = loff[l] + code_row0[(int64_t)l * num_views + v];
    try {
        DeviceGuard dg(h->device);
        // ---- codes: copy every level into the combined table + validate + truncate
        // (Algorithm 1 per-pixel TopK)
        if (total_rows > 0) {
            const size_t nslots = (size_t)(total_rows * S);
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
            for (int l = 0; l < nlev; l++) {
                if (rows[l] == 0) continue;
                if (!dense)
                    CK(cudaMemcpyAsync(h->code_atoms_in + loff[l] * S, code_atoms[l], sizeof(uint32_t) * rows[l] * S,
                                       cudaMemcpyDefault, h->stream));
                CK(cudaMemcpyAsync(h->code_coefs_in + loff[l] * S, code_coefs[l], sizeof(float) * rows[l] * S,
                                   cudaMemcpyDefault, h->stream));
            }
            if (dense)
                launch_ingest_dense(h->code_coefs_in, total_rows * S, h->code_coefs, latch_of(h), h->stream);
            else
                launch_ingest_codes(h->code_atoms_in, h->code_coefs_in, total_rows, S, h->K, h->L, h->code_atoms,
                                    h->code_coefs, latch_of(h), h->stream);
        }
        CallArgs args{nullptr, bn, row0c.data(), num_regions, num_views, S, (long long*)contributions_out, npx,
                      dense};
        const scoup_status st = run_views(h, num_views, cameras, bn, npx, args, region_ids, nlev);
        h->kernel_launches += total_rows > 0 ? 1 : 0;
        if (st != SCOUP_OK) return st;
    } catch (const CudaError& e) {
        return fail(e.err == cudaErrorMemoryAllocation ? SCOUP_ENOMEM : SCOUP_ECUDA,
                    std::string("CUDA error in ") + e.where + ": " + cudaGetErrorString(e.err));
    }
    return SCOUP_OK;
}

scoup_status scoup_uplift_render_views(scoup_uplift* h, int32_t num_views, const scoup_camera* cameras,
                                       const uint32_t* code_atoms, const float* code_coefs, int32_t K, float* out) {
    g_last_error.clear();
    if (!h) return fail(SCOUP_EINVAL, "handle is NULL");
    if (h->latched) return fail(SCOUP_ESTATE, "a latched data error is pending; call scoup_uplift_reset");
    if (num_views < 0) return fail(SCOUP_EINVAL, "num_views < 0");
    if (num_views == 0) return SCOUP_OK;
    if (!cameras || !code_atoms || !code_coefs || !out) return fail(SCOUP_EINVAL, "NULL argument");
    if (K < 1 || K > SCOUP_MAX_K) return fail(SCOUP_EINVAL, "K out of range");
    if (h->L > 128) return fail(SCOUP_EUNSUPPORTED, "render needs L <= 128 (per-pixel rows in shared memory)");
    if (!is_device_ptr(code_atoms) || !is_device_ptr(code_coefs) || !is_device_ptr(out))
        return fail(SCOUP_EINVAL, "render buffers must be device memory");
    const int Wd = cameras[0].width, Hd = cameras[0].height;
    for (int v = 0; v < num_views; v++) {
        const scoup_camera& c = cameras[v];
        if (c.width != Wd || c.height != Hd) return fail(SCOUP_EINVAL, "cameras of one call must share width/height");
        if (c.width <= 0 || c.height <= 0) return fail(SCOUP_EINVAL, "camera width/height <= 0");
        if (!(c.fx > 0.f) || !(c.fy > 0.f) || !std::isfinite(c.fx) || !std::isfinite(c.fy) || !std::isfinite(c.cx) ||
            !std::isfinite(c.cy))
            return fail(SCOUP_EINVAL, "camera " + std::to_string(v) + ": bad intrinsics");
        if (!rigid_ok(c.world_to_camera))
            return fail(SCOUP_EDATA, "camera " + std::to_string(v) + ": world_to_camera is not rigid (1e-5)");
    }
    if ((int64_t)Wd * Hd >= (int64_t)INT32_MAX) return fail(SCOUP_EUNSUPPORTED, "image too large");
    if ((int64_t)((Wd + TILE - 1) / TILE + 1) * ((Hd + TILE - 1) / TILE + 1) > MAX_SAT_ENTRIES)
        return fail(SCOUP_EUNSUPPORTED, "image too large for the tile tables (> 12288 16x16 tiles)");
    const int64_t npx = (int64_t)Wd * Hd;
    DeviceGuard dg(h->device);
    if (h->G == 0) {
        try {
            CK(cudaMemsetAsync(out, 0, sizeof(float) * npx * h->L * num_views, h->stream));
        } catch (const CudaError& e) {
            return fail(SCOUP_ECUDA, std::string("CUDA error in ") + e.where + ": " + cudaGetErrorString(e.err));
        }
        return SCOUP_OK;
    }
    const Binning bn = choose_binning(Wd, Hd, h->bin_shift);
    CallArgs args{nullptr, bn, nullptr, nullptr, num_views, 1, nullptr, npx, false};
    args.render = true;
    args.r_atoms = code_atoms;
    args.r_coefs = code_coefs;
    args.rK = K;
    args.r_out = out;
    return run_views(h, num_views, cameras, bn, npx, args, nullptr, 0);
}

scoup_status scoup_uplift_decode(scoup_uplift* h, int64_t num_pixels, const float* W_hat, const float* C, int32_t D,
                                 float* F) {
    g_last_error.clear();
    if (!h) return fail(SCOUP_EINVAL, "handle is NULL");
    if (num_pixels < 0 || D < 1) return fail(SCOUP_EINVAL, "bad sizes");
    if (num_pixels == 0) return SCOUP_OK;
    if (!W_hat || !C || !F) return fail(SCOUP_EINVAL, "NULL argument");
    if (num_pixels > (int64_t)INT32_MAX) return fail(SCOUP_EUNSUPPORTED, "num_pixels >= 2^31");
    DeviceGuard dg(h->device);
    const char* mode = std::getenv("SCOUP_DECODE");  // "sgemm": the cuBLAS path (A/B measurements)
    if (decode_tc_supported(h->L, D) && !(mode && std::string(mode) == "sgemm")) {
        if (!is_device_ptr(W_hat) || !is_device_ptr(C) || !is_device_ptr(F))
            return fail(SCOUP_EINVAL, "decode buffers must be device memory");
        if ((reinterpret_cast<uintptr_t>(W_hat) | reinterpret_cast<uintptr_t>(F)) & 15)
            return fail(SCOUP_EINVAL, "W_hat / F must be 16-byte aligned");
        try {
            int sms = 0;
            CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, h->device));
            float* scratch = nullptr;
            dalloc(&scratch, decode_tc_scratch_bytes(h->L, D) / sizeof(float), h->stream);
            const cudaError_t le = launch_decode_tc(W_hat, num_pixels, h->L, D, C, scratch, F, sms, h->stream);
            if (le != cudaSuccess) throw CudaError{le, "launch_decode_tc"};
            h->kernel_launches += 2;
            dfree(scratch, h->stream);
        } catch (const CudaError& e) {
            return fail(e.err == cudaErrorMemoryAllocation ? SCOUP_ENOMEM : SCOUP_ECUDA,
                        std::string("CUDA error in ") + e.where + ": " + cudaGetErrorString(e.err));
        }
        return SCOUP_OK;
    }
    if (!h->blas) {
        if (cublasCreate(&h->blas) != CUBLAS_STATUS_SUCCESS) return fail(SCOUP_ECUDA, "cublasCreate failed");
    }
    cublasSetStream(h->blas, h->stream);
    cublasSetMathMode(h->blas, CUBLAS_PEDANTIC_MATH);  // fp32 throughout (no TF32)
    // row-major F [P, D] = W_hat [P, L] C [L, D]  <=>  column-major F^T = C^T W_hat^T
    const float one = 1.f, zero = 0.f;
    const cublasStatus_t st = cublasSgemm(h->blas, CUBLAS_OP_N, CUBLAS_OP_N, D, (int)num_pixels, h->L, &one, C, D,
                                          W_hat, h->L, &zero, F, D);
    if (st != CUBLAS_STATUS_SUCCESS) return fail(SCOUP_ECUDA, "cublasSgemm failed");
    return SCOUP_OK;
}

scoup_status scoup_uplift_finalize_topk(scoup_uplift* h, int64_t first_row, int64_t num_rows, const float* W_rows,
                                        const float* Z_rows, uint32_t* out_atoms, float* out_coefs) {
    return scoup_uplift_finalize_topk_level(h, 0, first_row, num_rows, W_rows, Z_rows, out_atoms, out_coefs);
}

scoup_status scoup_uplift_finalize_topk_level(scoup_uplift* h, int32_t level, int64_t first_row, int64_t num_rows,
                                              const float* W_rows, const float* Z_rows, uint32_t* out_atoms,
                                              float* out_coefs) {
    return scoup_uplift_finalize_topk_entropy(h, level, first_row, num_rows, W_rows, Z_rows, out_atoms, out_coefs,
                                              nullptr);
}

scoup_status scoup_uplift_finalize_topk_entropy(scoup_uplift* h, int32_t level, int64_t first_row, int64_t num_rows,
                                                const float* W_rows, const float* Z_rows, uint32_t* out_atoms,
                                                float* out_coefs, float* out_entropy) {
    g_last_error.clear();
    (void)Z_rows;
    if (!h) return fail(SCOUP_EINVAL, "handle is NULL");
    if (first_row < 0 || num_rows < 0) return fail(SCOUP_EINVAL, "negative row range");
    if (level < 0 || level >= h->nlev) return fail(SCOUP_EINVAL, "level out of range");
    if (num_rows > 0 && (!out_atoms || !out_coefs)) return fail(SCOUP_EINVAL, "NULL output");
    if (!W_rows && first_row + num_rows > h->Npad) return fail(SCOUP_EINVAL, "row range beyond rows_padded");
    try {
        DeviceGuard dg(h->device);
        // (checked before any allocation or event record below)
        if (num_rows > 0 && out_entropy && !is_device_ptr(out_entropy))
            return fail(SCOUP_EINVAL, "out_entropy must be device memory");
        if (num_rows > 0) {
            const float* Wsrc =
                W_rows ? W_rows : h->W + ((int64_t)level * h->Npad + first_row) * (int64_t)h->L;
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
            launch_topk(Wsrc, num_rows, valid, h->L, h->K, da, dc, out_entropy, h->stream);
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

scoup_status scoup_uplift_finalize_topk_peers(scoup_uplift* h, int32_t level, int64_t first_row, int64_t num_rows,
                                              int32_t num_peers, const float* const* W_peers, uint32_t* out_atoms,
                                              float* out_coefs) {
    g_last_error.clear();
    if (!h) return fail(SCOUP_EINVAL, "handle is NULL");
    if (first_row < 0 || num_rows < 0 || first_row + num_rows > h->Npad)
        return fail(SCOUP_EINVAL, "row range outside [0, rows_padded)");
    if (level < 0 || level >= h->nlev) return fail(SCOUP_EINVAL, "level out of range");
    if (num_peers < 1 || num_peers > MAX_PEERS) return fail(SCOUP_EINVAL, "num_peers outside [1, 16]");
    if (!W_peers) return fail(SCOUP_EINVAL, "W_peers is NULL");
    if (num_rows > 0 && (!out_atoms || !out_coefs)) return fail(SCOUP_EINVAL, "NULL output");
    if (h->L % 4 != 0) return fail(SCOUP_EUNSUPPORTED, "peer reduction needs L % 4 == 0");
    PeerRows pr{};
    pr.n = num_peers;
    for (int q = 0; q < num_peers; q++) {
        if (!W_peers[q] || (reinterpret_cast<uintptr_t>(W_peers[q]) & 15))
            return fail(SCOUP_EINVAL, "peer accumulator " + std::to_string(q) + " NULL or not 16-byte aligned");
        pr.W[q] = W_peers[q] + (int64_t)level * h->Npad * h->L;
    }
    try {
        DeviceGuard dg(h->device);
        if (num_rows > 0) {
            if (!is_device_ptr(out_atoms) || !is_device_ptr(out_coefs))
                return fail(SCOUP_EINVAL, "peer finalize writes device outputs");
            const int64_t valid = std::max<int64_t>(0, std::min<int64_t>(num_rows, h->G - first_row));
            launch_topk_peers(pr, first_row, num_rows, valid, h->L, h->K, out_atoms, out_coefs, h->stream);
            h->kernel_launches += 1;
            CK(cudaGetLastError());
        }
        CK(cudaStreamSynchronize(h->stream));
        return check_latched(h);
    } catch (const CudaError& e) {
        return fail(SCOUP_ECUDA, std::string("CUDA error in ") + e.where + ": " + cudaGetErrorString(e.err));
    }
}

scoup_status scoup_ipc_export(const void* dptr, void* handle_out, int64_t* offset_out) {
    g_last_error.clear();
    if (!dptr || !handle_out || !offset_out) return fail(SCOUP_EINVAL, "NULL argument");
    static CUresult (*range)(CUdeviceptr*, size_t*, CUdeviceptr) = nullptr;
    if (!range) {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q{};
        if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn)
            return fail(SCOUP_ECUDA, "cuMemGetAddressRange unavailable");
        range = reinterpret_cast<CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr)>(fn);
    }
    CUdeviceptr base = 0;
    size_t size = 0;
    if (range(&base, &size, reinterpret_cast<CUdeviceptr>(dptr)) != CUDA_SUCCESS)
        return fail(SCOUP_EINVAL, "not a device allocation");
    cudaIpcMemHandle_t hd;
    const cudaError_t e = cudaIpcGetMemHandle(&hd, reinterpret_cast<void*>(base));
    if (e != cudaSuccess) return fail(SCOUP_ECUDA, std::string("cudaIpcGetMemHandle: ") + cudaGetErrorString(e));
    static_assert(sizeof(cudaIpcMemHandle_t) == SCOUP_IPC_HANDLE_BYTES, "IPC handle size");
    std::memcpy(handle_out, &hd, sizeof(hd));
    *offset_out = (int64_t)(reinterpret_cast<CUdeviceptr>(dptr) - base);
    return SCOUP_OK;
}

scoup_status scoup_ipc_import(int device, const void* handle, int64_t offset, void** dptr_out, void** base_out) {
    g_last_error.clear();
    if (!handle || !dptr_out || !base_out || offset < 0) return fail(SCOUP_EINVAL, "bad argument");
    DeviceGuard dg(device);
    cudaIpcMemHandle_t hd;
    std::memcpy(&hd, handle, sizeof(hd));
    void* base = nullptr;
    const cudaError_t e = cudaIpcOpenMemHandle(&base, hd, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) return fail(SCOUP_ECUDA, std::string("cudaIpcOpenMemHandle: ") + cudaGetErrorString(e));
    *base_out = base;
    *dptr_out = static_cast<char*>(base) + offset;
    return SCOUP_OK;
}

scoup_status scoup_ipc_close(int device, void* base) {
    g_last_error.clear();
    if (!base) return SCOUP_OK;
    DeviceGuard dg(device);
    const cudaError_t e = cudaIpcCloseMemHandle(base);
    if (e != cudaSuccess) return fail(SCOUP_ECUDA, std::string("cudaIpcCloseMemHandle: ") + cudaGetErrorString(e));
    return SCOUP_OK;
}

scoup_status scoup_uplift_reset(scoup_uplift* h) {
    g_last_error.clear();
    if (!h) return fail(SCOUP_EINVAL, "handle is NULL");
    try {
        DeviceGuard dg(h->device);
        CK(cudaMemsetAsync(h->W, 0, sizeof(float) * std::max<int64_t>(1, h->Npad) * h->L * h->nlev, h->stream));
        CK(cudaMemsetAsync(h->Z, 0, sizeof(float) * std::max<int64_t>(1, h->Npad), h->stream));
        CK(cudaMemsetAsync(h->d_stats, 0, 6 * sizeof(unsigned long long), h->stream));
        CK(cudaMemsetAsync(h->d_err_code, 0, sizeof(int), h->stream));
        h->latched = false;
        h->host_entries = 0;
        h->kernel_launches = 0;
        h->cub_launches = 0;
        h->batches[0] = h->batches[1] = 0;
        h->near_frac_changes = 0;
        h->host_map_chunks = 0;
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
        unsigned long long s[6];
        CK(cudaStreamSynchronize(h->stream));
        CK(cudaMemcpy(s, h->d_stats, sizeof(s), cudaMemcpyDeviceToHost));
        out->views = (int64_t)s[0];
        out->contributions = (int64_t)s[1];
        out->tile_entries = h->host_entries;
        out->visible = (int64_t)s[3];
        out->support_tests = (int64_t)s[4];
        out->kernel_launches = h->kernel_launches;
        out->cub_launches = h->cub_launches;
        out->lane_evaluations = (int64_t)s[5];
        out->global_reds = (int64_t)s[2];
        out->view_batch = MAX_VB;
        out->batches[0] = h->batches[0];
        out->batches[1] = h->batches[1];
        out->near_frac_changes = h->near_frac_changes;
        out->host_map_chunks = h->host_map_chunks;
        out->near_frac = h->near_frac;
        return check_latched(h);
    } catch (const CudaError& e) {
        return fail(SCOUP_ECUDA, std::string("CUDA error in ") + e.where + ": " + cudaGetErrorString(e.err));
    }
}

scoup_status scoup_uplift_set_counters(scoup_uplift* h, int enable) {
    g_last_error.clear();
    if (!h) return fail(SCOUP_EINVAL, "handle is NULL");
    h->count_tests = enable != 0;
    return SCOUP_OK;
}

scoup_status scoup_uplift_set_pipeline(scoup_uplift* h, int contexts) {
    g_last_error.clear();
    if (!h) return fail(SCOUP_EINVAL, "handle is NULL");
    if (contexts != 1 && contexts != 2) return fail(SCOUP_EINVAL, "contexts must be 1 or 2");
    h->nctx = contexts;
    return SCOUP_OK;
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
    void* ptrs[] = {h->pg.a, h->pg.b, h->pg.c, h->pg.s2, h->d_err_code, h->d_err_index, h->d_stats, h->code_atoms,
                    h->code_coefs, h->code_atoms_in, h->code_coefs_in};
    for (void* p : ptrs) dfree(p, h->stream);
    if (h->own_wz) {
        dfree(h->W, h->stream);
        dfree(h->Z, h->stream);
    }
    if (h->blas) cublasDestroy(h->blas);
    dfree(h->ids_all, h->stream);
    cudaStreamSynchronize(h->stream);
    if (h->copy_s) {
        cudaStreamSynchronize(h->copy_s);
        cudaStreamDestroy(h->copy_s);
    }
    for (cudaEvent_t e : h->chunk_ev) cudaEventDestroy(e);
    delete h;
}

}  // extern "C"
