/*
 * scoup_diag.h -- measurement helpers of libscoup.so (not part of the method's API).
 *
 * SURVEY.md §8(d) asks for the fused kernel's scatter-add (Algorithm 1 line 9, P:360:
 * W[i][a] += c e; Eq. 5) to be reported against a MEASURED L2 atomic-reduction
 * throughput R_red, since the B200's datasheets give none.  bench.py calls this once per run.
 */
#ifndef SCOUP_DIAG_H
#define SCOUP_DIAG_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Throughput of `red.global.add.f32` (vec4 = 0) or `red.global.v4.f32.add` (vec4 = 1) on
 * device `device`: a buffer of buffer_bytes (>= 4096; 32 MB stays L2-resident, 4 GB does not) is
 * allocated and zeroed, then `launches` launches of 8 CTAs x 256 threads per SM issue about
 * reds_per_launch float adds each, to distinct addresses: consecutive floats per warp
 * (scattered = 0) or one 32-byte sector per lane at hashed positions (scattered = 1).
 * Out: *adds_per_s = float adds per second (CUDA events around the timed launches, after one
 * warm-up launch); *ms_per_launch (may be NULL).  The buffer is freed before returning.
 * Returns 0, 1 (bad argument) or 3 (CUDA error; scoup_diag_last_error() has the text).
 * Synchronous; uses the legacy default stream of the calling thread. */
int scoup_diag_red_rate(int device, int64_t buffer_bytes, int scattered, int vec4, int64_t reds_per_launch,
                        int launches, double *adds_per_s, double *ms_per_launch);

/* Entries per warp segment of the binning's stable counting sort (DESIGN.md §5 a3; process-wide):
 * entries_per_segment > 0 forces that length (rounded up to a multiple of 32; tests use it to
 * exercise the long segments large chunks get), 0 restores the adaptive choice (2048 entries, more
 * for chunks so large that the [segment][bin] count matrix would dominate).  Returns 0, or 1 if
 * entries_per_segment is negative or above 2^24. */
int scoup_diag_set_binsort_segment(int entries_per_segment);

/* Region slots per 16x16 tile of the fused raster kernel (DESIGN.md §5 a4; process-wide): the
 * kernel exists with 4 and with 8 shared-sum slots (tiles meeting more regions aggregate per
 * pixel); 0 restores the adaptive choice (4 when every view of the batch averages >= 64 x 64 px
 * per region, else 8), 4 or 8 forces a variant (tests: both variants on every configuration).
 * Returns 0, or 1 for any other value. */
int scoup_diag_set_raster2_slots(int slots);

/* Thread-local message of the last failing diag call ("" if none). */
const char *scoup_diag_last_error(void);

#ifdef __cplusplus
}
#endif

#endif /* SCOUP_DIAG_H */
