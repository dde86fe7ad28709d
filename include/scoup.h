/*
 * scoup.h -- C ABI of the B200-native weighted sparse aggregation library (libscoup.so).
 *
 * SCOUP (arXiv 2605.13600) "sparse coefficient uplifting": for every view v, a forward
 * pass of the 3DGS rasteriser yields the blending weights e_i(v,p) = alpha_i prod_{j<i}
 * (1-alpha_j) (Eq. 2).  Each pixel's region sparse code W_v(p) (<= S
 * (atom, coef) pairs over L atoms, Eq. 4) is scaled by e and scatter-added into a
 * per-Gaussian L-vector (Eq. 5; Algorithm 1), together with the weight
 * sum Z_i (Eq. 3).  After all views, every Gaussian keeps its Top-K atoms,
 * L1-renormalised (Eq. 6; Algorithm 1).
 *
 * The fragment weights follow the reproducible fp32 arithmetic of DESIGN.md §3, so they
 * are bit-identical to the CPU oracle's; only the summation order of W and Z differs.
 *
 * Conventions (all entry points):
 *  - Every call is stream-ordered on the stream given to scoup_uplift_init (a cudaStream_t
 *    passed as void*; NULL = legacy default stream).  Calls return once work is enqueued,
 *    except where noted ("synchronises").
 *  - Array arguments marked "device or host" may point to device memory or to host memory
 *    (pinned or pageable); host arrays are copied to the device inside the call, on the
 *    handle's stream, before it returns (so the caller may reuse them on return).  Device
 *    arrays must stay valid until the stream reaches the call (CUDA-API style).
 *  - Ownership: the caller owns every buffer it passes.  The handle owns its scratch and, if
 *    W/Z were NULL at init, its accumulators (freed by scoup_uplift_free).
 *  - Errors: return codes only; nothing is thrown across the ABI.  Host-checkable problems
 *    return immediately and leave the handle unchanged.  Problems found on the device
 *    (non-finite Gaussian, region id >= R_v, atom >= L, negative/non-finite coef) are
 *    latched in the handle and returned (SCOUP_EDATA) by the next synchronising call;
 *    accumulators are undefined afterwards until scoup_uplift_reset.
 *    scoup_last_error() returns a thread-local message naming the offending index.
 *  - The handle is not thread-safe; use one handle per (device, semantic level).
 */
#ifndef SCOUP_H
#define SCOUP_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SCOUP_NONE 0xFFFFFFFFu  /* unassigned pixel / empty code slot */
#define SCOUP_MAX_L 1024        /* implementation limits (EUNSUPPORTED beyond) */
#define SCOUP_MAX_K 32
#define SCOUP_MAX_S 16          /* per call: num_levels * S <= SCOUP_MAX_S */
#define SCOUP_MAX_LEVELS 4

typedef struct scoup_uplift scoup_uplift; /* opaque */

typedef enum {
    SCOUP_OK = 0,
    SCOUP_EINVAL = 1,       /* bad argument / configuration (e.g. K > L) */
    SCOUP_EDATA = 2,        /* bad input data (non-finite, bad id, non-rigid camera) */
    SCOUP_ECUDA = 3,        /* CUDA runtime failure (message has cudaGetErrorString) */
    SCOUP_ENOMEM = 4,       /* device allocation failed */
    SCOUP_ESTATE = 5,       /* call not valid in the handle's state */
    SCOUP_EUNSUPPORTED = 6  /* beyond SCOUP_MAX_L / _K / _S or too many pixels */
} scoup_status;

/* Pinhole camera, no distortion, OpenCV axes (+x right, +y down, +z forward).
 * world_to_camera: row-major 4x4 rigid transform [R|t; 0 0 0 1] ("camera pose"). */
typedef struct {
    float fx, fy, cx, cy;
    int32_t width, height;
    float world_to_camera[16];
} scoup_camera;

/* Counters accumulated since init / the last reset (read by scoup_uplift_get_stats). */
typedef struct {
    int64_t views;          /* views added */
    int64_t contributions;  /* fragments (v,p,i) with e > 0: terms of Eq. 5's sum; counted
                               while scoup_uplift_set_counters(h, 1) is on or for calls given a
                               contributions_out array */
    int64_t tile_entries;   /* (Gaussian, tile) pairs binned */
    int64_t visible;        /* sum over views of Gaussians passing the projection culls */
    int64_t support_tests;  /* (pixel, Gaussian) pairs inside the Gaussian's square support
                               tested while the pixel was still active (Eq. 2 work); counted
                               only while scoup_uplift_set_counters(h, 1) is on */
    int64_t kernel_launches;/* launches of this library's own kernels (CUB sort/scan excluded) */
    int64_t cub_launches;   /* CUB device-wide sort/scan calls */
    int64_t lane_evaluations; /* lanes that ran the per-pixel sequence on a record (32 per
                                 (warp, record) evaluated; counted with the support tests):
                                 support_tests / lane_evaluations is the raster's lane use */
    int64_t batches[2];     /* view batches run by each of the two pipeline contexts */
    int64_t near_frac_changes; /* in-call adaptations of the near-chunk fraction (DESIGN.md §5 a3) */
    int64_t host_map_chunks;/* up-front host->device region-map copy chunks (host region_ids) */
    double near_frac;       /* the near-chunk fraction now in use */
    int64_t global_reds;    /* red.global.add.f32 issued by the fused kernel's flush into W and Z
                               (lane level; counted with the support tests) */
    int64_t view_batch;     /* views per pipeline batch (the library's batch size) */
} scoup_stats;

/* Per-kernel-class device time (CUDA events on the launching streams), accumulated while
 * timing is enabled.  Milliseconds. */
typedef struct {
    double preprocess_ms;   /* preprocess + depth sort + tile-count scan (stage 1) */
    double binning_ms;      /* entry emission + tile sort + ranges (stage 2 front) */
    double raster_ms;       /* fused rasterise-and-aggregate kernel */
    double topk_ms;         /* finalize Top-K kernel */
    int64_t raster_launches;
    int64_t views_timed;
} scoup_timing;

/*
 * Create an uplift handle for one semantic level on `device`.
 *  num_gaussians  N >= 0 (0 allowed: every later call is a no-op producing nothing).
 *  means [N,3], scales [N,3] (activated, > 0), rotations [N,4] (w,x,y,z; normalised
 *  inside), opacities [N] (activated, in [0,1]) -- float32, device or host.  The handle
 *  derives its own packed copy (activation + Sigma_3D, DESIGN.md §3 G1), so the inputs may
 *  be freed once the call returns (host) / the stream passes it (device).
 *  L  number of codebook atoms (1..SCOUP_MAX_L); K  output Top-K (1..min(L, SCOUP_MAX_K)).
 *  W [rows_padded, L] / Z [rows_padded] float32 device accumulators, zeroed here; NULL ->
 *  the handle allocates them.  rows_padded >= N (e.g. a multiple of the rank count so that
 *  a reduce-scatter can split them); 0 -> N.
 *  Errors: EINVAL (null out / negative N / K < 1 / K > L / rows_padded < N), EUNSUPPORTED,
 *  ENOMEM, ECUDA.  Non-finite means/scales/rotations or opacity outside [0,1] are latched
 *  (EDATA at the next synchronising call).
 */
scoup_status scoup_uplift_init(int device, void *cuda_stream, int64_t num_gaussians,
                               const float *means, const float *scales, const float *rotations,
                               const float *opacities, int32_t L, int32_t K, float *W, float *Z,
                               int64_t rows_padded, scoup_uplift **out);

/*
 * Fused multi-level uplift.  The paper uplifts its three SAM levels
 * (fine / medium / coarse) independently and renders them together; every level
 * sees exactly the same fragments e_i(v,p) -- only the region maps and codes differ -- so one
 * projection, sort and raster pass can feed all of them.  A handle made here holds num_levels
 * accumulators: W [num_levels, rows_padded, L] (level-major, contiguous; caller-allocated or
 * NULL) and one Z [rows_padded] (Z_i counts every fragment, whatever the region, so it is the
 * same for all levels).  num_levels in 1..SCOUP_MAX_LEVELS; scoup_uplift_init is this with 1.
 * Other arguments and errors as scoup_uplift_init.
 */
scoup_status scoup_uplift_init_levels(int device, void *cuda_stream, int64_t num_gaussians,
                                      const float *means, const float *scales, const float *rotations,
                                      const float *opacities, int32_t num_levels, int32_t L, int32_t K,
                                      float *W, float *Z, int64_t rows_padded, scoup_uplift **out);

/*
 * Rasterise `num_views` views and scatter-add their sparse codes (Eq. 5 / Algorithm 1
 * lines 5-12) into the handle's accumulators.  May be called any number of times.
 *  cameras      host [V]; all views of one call must share width/height.
 *  region_ids   [V,H,W] uint32, device or host: region of each pixel, SCOUP_NONE = none.
 *               Pixels with SCOUP_NONE add to Z but not to W.
 *  code_row0    host [V]: first row of view v's codes in code_atoms/code_coefs.
 *  num_regions  host [V]: R_v; ids must be < R_v (else latched EDATA).
 *  code_atoms   [rows,S] uint32, code_coefs [rows,S] float32, device or host
 *               (rows = max_v code_row0[v] + num_regions[v]); SCOUP_NONE = empty slot;
 *               coefficients finite and >= 0.  A code with more than K filled slots is
 *               truncated to its K largest (Algorithm 1's per-pixel TopK).
 *               code_atoms NULL: DENSE region features (the dense feature uplift of Eq. 3,
 *               P:76-80, the baseline SCOUP replaces): S must equal L, code_coefs holds each
 *               region's full L-vector (any finite values), slot s adds to W[i][s]; no
 *               truncation.  W / Z then gives Eq. 3's f_i.
 *  contributions_out  optional device int64 [V]: per-view contribution counts are ADDED.
 *  Errors: EINVAL (null pointers, V < 0, S < 1, size mismatch, bad camera intrinsics),
 *  EDATA (camera rotation not orthonormal with det +1 within 1e-5), EUNSUPPORTED (S >
 *  SCOUP_MAX_S, H*W >= 2^31), ESTATE (latched error pending), ENOMEM, ECUDA.
 */
scoup_status scoup_uplift_add_views(scoup_uplift *h, int32_t num_views, const scoup_camera *cameras,
                                    const uint32_t *region_ids, const int64_t *code_row0,
                                    const int32_t *num_regions, const uint32_t *code_atoms,
                                    const float *code_coefs, int32_t S, int64_t *contributions_out);

/*
 * scoup_uplift_add_views for a handle of num_levels levels (scoup_uplift_init_levels):
 *  region_ids   host array of num_levels pointers, each [V,H,W] (device or host, as above);
 *  code_row0    host [num_levels, V]; num_regions host [num_levels, V];
 *  code_atoms / code_coefs  host arrays of num_levels pointers to each level's code table.
 *  num_levels * S <= SCOUP_MAX_S.  A region-id data error names the level.
 *  scoup_uplift_add_views is this with one level (ESTATE on a multi-level handle).
 */
scoup_status scoup_uplift_add_views_levels(scoup_uplift *h, int32_t num_views, const scoup_camera *cameras,
                                           const uint32_t *const *region_ids, const int64_t *code_row0,
                                           const int32_t *num_regions, const uint32_t *const *code_atoms,
                                           const float *const *code_coefs, int32_t S, int64_t *contributions_out);

/*
 * Eq. 6 on rows [first_row, first_row + num_rows): per Gaussian, order the accumulated
 * coefficients by (value desc, atom asc), keep the first K positive ones, divide by their
 * sum (Z_i cancels) and pad with (SCOUP_NONE, 0).  A row with W_i == 0 gives an
 * empty code (Algorithm 1 line 15).  Rows >= N (padding) give empty codes.
 *  W_rows [num_rows,L], Z_rows [num_rows] device: NULL -> the handle's own accumulators;
 *  else an externally reduced shard (e.g. the output of an NCCL reduce-scatter).
 *  out_atoms [num_rows,K] uint32, out_coefs [num_rows,K] float32: device or host (host:
 *  copied back, the call then synchronises).
 *  Synchronises the stream to report latched device errors (EDATA).
 *  Accumulators are not consumed: more views may follow and finalize may be re-run.
 */
scoup_status scoup_uplift_finalize_topk(scoup_uplift *h, int64_t first_row, int64_t num_rows,
                                        const float *W_rows, const float *Z_rows,
                                        uint32_t *out_atoms, float *out_coefs);

/*
 * Sparse coefficient rendering (Eq. 7):
 *   W_hat_v(p) = sum_{i in N_{v,p}} w_hat_i e_i(v,p)
 * for each view, with the handle's Gaussians and the K-sparse codes w_hat_i (the output of
 * scoup_uplift_finalize_topk: code_atoms [N,K] uint32 / code_coefs [N,K] float32, device;
 * SCOUP_NONE slots ignored).  e_i(v,p) are the same fragment weights as the uplift's
 * (bit-identical to the oracle's).  out: device float32 [V, H, W, L] (row-major, a dense
 * L-vector per pixel), overwritten.  L <= 128.  Stream-ordered; accumulators untouched.
 * Errors: EINVAL (NULL / host buffers, K out of range, camera problems as add_views), EDATA
 * (non-rigid camera), EUNSUPPORTED (L > 128, image too large), ECUDA.
 */
scoup_status scoup_uplift_render_views(scoup_uplift *h, int32_t num_views, const scoup_camera *cameras,
                                       const uint32_t *code_atoms, const float *code_coefs, int32_t K, float *out);

/*
 * Codebook decode (Eq. 8): F = W_hat C for num_pixels rendered coefficient
 * vectors W_hat [P, L] (e.g. scoup_uplift_render_views' output) and a codebook C [L, D], all
 * float32 row-major on the device; F [P, D] overwritten; W_hat and F 16-byte aligned.  With
 * L % 8 == 0, L <= 64 and D % 64 == 0 it runs the library's tcgen05 kernel (3xTF32: every
 * operand split exactly into a tf32 head and tail, fp32 accumulation in tensor memory, accuracy
 * of an fp32 GEMM); other shapes use cuBLAS SGEMM (fp32, no TF32).  SCOUP_DECODE=sgemm forces
 * the cuBLAS path (measurement only).  Stream-ordered on the handle's stream; a scratch of
 * 8 L D bytes comes from the stream-ordered pool.  Non-finite inputs give non-finite outputs.
 * Errors: EINVAL (NULL / host buffers, misaligned, bad sizes), EUNSUPPORTED (P >= 2^31),
 * ENOMEM, ECUDA.
 */
scoup_status scoup_uplift_decode(scoup_uplift *h, int64_t num_pixels, const float *W_hat, const float *C, int32_t D,
                                 float *F);

/* scoup_uplift_finalize_topk on level `level` (0 .. num_levels-1) of a multi-level handle;
 * scoup_uplift_finalize_topk is level 0.  EINVAL for a level out of range. */
scoup_status scoup_uplift_finalize_topk_level(scoup_uplift *h, int32_t level, int64_t first_row, int64_t num_rows,
                                              const float *W_rows, const float *Z_rows, uint32_t *out_atoms,
                                              float *out_coefs);

/*
 * finalize_topk_level plus, per row, the entropy of the Gaussian's aggregated coefficient
 * distribution before Top-K: with
 * w_l = W_l / sum_l W_l (Z cancels; negative-free by construction),
 * H = -sum_l w_l ln w_l, computed in the same pass over the row (fp32; NaN for W_i == 0).
 * out_entropy: device float [num_rows] (NULL = none).  Otherwise as finalize_topk_level.
 */
scoup_status scoup_uplift_finalize_topk_entropy(scoup_uplift *h, int32_t level, int64_t first_row, int64_t num_rows,
                                                const float *W_rows, const float *Z_rows, uint32_t *out_atoms,
                                                float *out_coefs, float *out_entropy);

/*
 * Fused cross-rank reduction + Top-K (Eq. 5 is a sum over views, so
 * the ranks' view-sharded partials add; Eq. 6, on the sum).  Rows [first_row,
 * first_row + num_rows) of level `level`: W = sum over q < num_peers of W_peers[q] (summed in
 * rank order 0..P-1, fp32), then Top-K + L1 renormalisation exactly as
 * scoup_uplift_finalize_topk.  W_peers: host array of num_peers (<= 16) device-accessible
 * pointers to each rank's accumulator base (the W of scoup_uplift_init, [levels][rows_padded][L],
 * same layout on every rank): the local one and the others' CUDA IPC mappings
 * (scoup_ipc_import); 16-byte aligned; L % 4 == 0.  This replaces the reduce-scatter + finalize
 * pair: the shard's rows are read once, directly from the peers' memory over NVLink, and no
 * reduced shard is written.  The caller must ensure every peer's accumulation is complete
 * before the call and that no peer modifies or frees its W until every rank has returned
 * (e.g. a barrier on each side).  Outputs are device memory.  Synchronising.  Errors: EINVAL,
 * EUNSUPPORTED (L % 4 != 0), ECUDA.
 */
scoup_status scoup_uplift_finalize_topk_peers(scoup_uplift *h, int32_t level, int64_t first_row, int64_t num_rows,
                                              int32_t num_peers, const float *const *W_peers, uint32_t *out_atoms,
                                              float *out_coefs);

/*
 * CUDA IPC plumbing for scoup_uplift_finalize_topk_peers: export a device pointer as an
 * allocation handle (SCOUP_IPC_HANDLE_BYTES opaque bytes) plus the pointer's offset inside that
 * allocation; import a peer's handle on `device` (peer access enabled lazily) -> the mapped
 * pointer and the mapping's base; close a mapping by its base.  The allocation must come from
 * cudaMalloc (e.g. the PyTorch caching allocator), not from a stream-ordered pool.
 */
#define SCOUP_IPC_HANDLE_BYTES 64
scoup_status scoup_ipc_export(const void *dptr, void *handle_out, int64_t *offset_out);
scoup_status scoup_ipc_import(int device, const void *handle, int64_t offset, void **dptr_out, void **base_out);
scoup_status scoup_ipc_close(int device, void *base);

/* Zero the accumulators and counters and clear a latched error (stream-ordered). */
scoup_status scoup_uplift_reset(scoup_uplift *h);

/* Device pointers of the accumulators: W [num_levels, rows_padded, L], Z [rows_padded] (Eq. 5
 * sums without 1/Z_i, and Z_i of Eq. 3).  Any out-pointer may be NULL. */
scoup_status scoup_uplift_get_accumulators(scoup_uplift *h, float **W, float **Z, int64_t *rows_padded);

/* Copy the counters (synchronises the stream; returns latched EDATA if any). */
scoup_status scoup_uplift_get_stats(scoup_uplift *h, scoup_stats *out);

/* Enable (1) / disable (0) the instrumented fused kernel, which counts contributions and support
 * tests (scoup_stats); off by default (the production kernel keeps no counters).  A call to
 * add_views with a contributions_out array always uses the instrumented kernel. */
scoup_status scoup_uplift_set_counters(scoup_uplift *h, int enable);

/* Number of pipeline contexts add_views alternates between: 2 (the default)
 * overlaps one view batch's front (depth pass, selection, sorts) with the other's raster; 1 runs
 * every step of every batch in order on one stream, so that per-kernel event times are each
 * kernel's own duration (bench.py's roofline timing pass).  Results are identical.  EINVAL
 * outside {1, 2}. */
scoup_status scoup_uplift_set_pipeline(scoup_uplift *h, int contexts);

/* Enable (1) / disable (0) per-kernel-class event timing; enabling clears the totals. */
scoup_status scoup_uplift_set_timing(scoup_uplift *h, int enable);

/* Totals since timing was enabled (synchronises the handle's streams). */
scoup_status scoup_uplift_get_timing(scoup_uplift *h, scoup_timing *out);

/* Release the handle (synchronises its stream).  NULL is a no-op. */
void scoup_uplift_free(scoup_uplift *h);

/* Thread-local message of the last failing call on this thread ("" if none). */
const char *scoup_last_error(void);

/* Library version string. */
const char *scoup_version(void);

#ifdef __cplusplus
}
#endif

#endif /* SCOUP_H */
