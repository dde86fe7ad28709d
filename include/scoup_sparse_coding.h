/*
 * scoup_sparse_coding.h -- C ABI of the 2D sparse coding step that produces SCOUP's region codes
 * (Eq. 4; recipe P:97 and P:158).  Same library as
 * scoup.h (libscoup.so); status codes and scoup_last_error() are shared.
 *
 * Problem (Eq. 4): R region features f_r in R^D (one per SAM region) are approximated as
 * f_r ~ w_r C with a codebook C in R^{L x D} and K-sparse convex codes w_r (||w_r||_0 <= K,
 * w_r >= 0, 1^T w_r = 1).  Method (DESIGN.md §14 readings R-SC1..R-SC7):
 *   w_r = soft_topk(z_r, K): softmax of the learnable logits z_r restricted to their K largest
 *         entries (ties -> lower index) and renormalised;
 *   loss = (1/R) sum_r (1 - cos(w_r C, f_r));
 *   full-batch Adam on (Z, C), gradients only through the kept support; codebook initialised
 *   by k-means (k-means++ seeding, Lloyd iterations) and logits by 10 cos(f_r, C_l).
 * The hard codes (scoup_sc_encode) are the code table scoup_uplift_add_views consumes (S = K).
 *
 * Everything runs on the device on the handle's stream; all float data are float32.
 * Limits: 1 <= K <= min(L, 32), L <= 128, D <= 1024, L * D <= 49152 (the per-CTA gradient
 * accumulator lives in shared memory), R >= 1.
 */
#ifndef SCOUP_SPARSE_CODING_H
#define SCOUP_SPARSE_CODING_H

#include <stdint.h>

#include "scoup.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct scoup_sc scoup_sc; /* opaque: one sparse-coding problem on one device */

/* Create a problem.  features: device [R, D] row-major, borrowed (must stay valid and
 * unchanged for the handle's lifetime); rows must be finite and non-zero (checked, latched
 * EDATA reported by the next synchronising call).  The handle owns C [L, D], Z [R, L] and the
 * Adam moments (all zero; t = 0).  Errors: EINVAL (NULL, bad sizes), EUNSUPPORTED (limits
 * above), ENOMEM, ECUDA. */
scoup_status scoup_sc_init(int device, void *cuda_stream, int64_t R, int32_t D, int32_t L, int32_t K,
                           const float *features, scoup_sc **out);

/* k-means initialisation (R-SC6): k-means++ seeding driven by the caller's draws --
 * uniforms: host [L] doubles in [0, 1); fallback: host [L, D] unit vectors used for atoms with
 * no distinct row left -- then Lloyd iterations (nearest centre, ties -> lower index; empty
 * clusters keep their centre) until the assignment is a fixpoint or max_iter.  Then
 * Z = 10 cos(f_r, C_l) (R-SC5), Adam moments = 0, t = 0.  iters_out (host, may be NULL): Lloyd
 * iterations run.  Synchronising.  Errors: EINVAL, ECUDA, EDATA (latched feature error). */
scoup_status scoup_sc_kmeans(scoup_sc *h, const double *uniforms, const float *fallback, int32_t max_iter,
                             int32_t *iters_out);

/* Overwrite the optimiser state (device pointers, NULL = leave as is): C [L, D], Z [R, L],
 * mC, vC [L, D], mZ, vZ [R, L], and the number of Adam steps already taken t >= 0.  Used to
 * resume training and by the parity tests (one epoch from a given state).  Stream-ordered. */
scoup_status scoup_sc_set_state(scoup_sc *h, const float *C, const float *Z, const float *mC, const float *vC,
                                const float *mZ, const float *vZ, int64_t t);

/* Device pointers to the handle's state (owned by the handle) and the step count. */
scoup_status scoup_sc_get_state(scoup_sc *h, float **C, float **Z, float **mC, float **vC, float **mZ,
                                float **vZ, int64_t *t);

/* `epochs` full-batch Adam epochs (lr, beta1, beta2, eps as in PyTorch; the paper: 4,000 epochs,
 * lr 7e-4).  Each epoch evaluates the loss and gradients at the current (Z, C) for all
 * regions, then updates Z and C with bias-corrected Adam at step t + 1.  loss_out (host or device
 * [epochs], may be NULL): the loss at the start of each epoch.  The epochs are replayed from a
 * captured CUDA graph.  Synchronising when loss_out is host memory.  Errors: EINVAL, EDATA
 * (non-finite loss: latched, with the epoch index), ECUDA. */
scoup_status scoup_sc_train(scoup_sc *h, int32_t epochs, float lr, float beta1, float beta2, float eps,
                            float *loss_out);

/* Hard codes (R-SC7): for each region its K kept atoms in logit order (ties -> lower index) and
 * their soft top-K weights.  atoms: device uint32 [R, K]; coefs: device float32 [R, K]. */
scoup_status scoup_sc_encode(scoup_sc *h, uint32_t *atoms, float *coefs);

void scoup_sc_free(scoup_sc *h);

#ifdef __cplusplus
}
#endif

#endif /* SCOUP_SPARSE_CODING_H */
