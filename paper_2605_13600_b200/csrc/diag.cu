// diag.cu -- measurement helpers behind include/scoup_diag.h (not part of the method).
//
// R_red: the L2 atomic-reduction throughput that SURVEY.md §8(d) names as the denominator of
// the fused kernel's scatter-add (Algorithm 1 line 9: W[i][a] += c e).  Every thread
// issues `red.global.add.f32` (or the v4 form, REDG.E.ADD.F32x4) to distinct addresses of a
// buffer that is either L2-resident (32 MB) or HBM-resident (4 GB), in one of two address
// patterns:
//   coalesced  lane l of a warp hits float l of a 128-B line (4 sectors per warp instruction);
//   scattered  every lane hits its own 32-B sector, lines spread over the buffer (the fused
//              kernel's flush pattern: S atoms of a 64-float W row per (slot, Gaussian), rows
//              of unrelated Gaussians in neighbouring lanes).
// The rate is float adds per second (4 per thread-instruction for v4), CUDA events around
// `iters` back-to-back launches after one warm-up launch.
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "../../include/scoup_diag.h"
#include "internal.cuh"

namespace {

template <bool V4, bool SCATTER>
__global__ void __launch_bounds__(256) red_kernel(float* buf, uint64_t nfloat, int per_thread, uint32_t salt) {
    const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const uint64_t nthreads = (uint64_t)gridDim.x * blockDim.x;
    const float v = 1.0f;
    for (int k = 0; k < per_thread; k++) {
        const uint64_t i = tid + (uint64_t)k * nthreads;
        uint64_t off;
        if (SCATTER) {
            // one 32-B sector per lane: sector index by a multiplicative hash of i
            const uint64_t nsec = nfloat / 8;
            const uint64_t sec = ((i + salt) * 0x9E3779B97F4A7C15ull >> 20) % nsec;
            off = sec * 8 + (V4 ? 4 * (i & 1) : (i & 7));
        } else {
            off = (V4 ? 4 * i : i) % (nfloat - (V4 ? 4 : 1));
            if (V4) off &= ~3ull;
        }
        float* p = buf + off;
        if (V4)
            asm volatile("red.global.v4.f32.add [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(v), "f"(v), "f"(v), "f"(v)
                         : "memory");
        else
            asm volatile("red.global.add.f32 [%0], %1;" ::"l"(p), "f"(v) : "memory");
    }
}

thread_local std::string g_diag_error;

}  // namespace

extern "C" {

const char* scoup_diag_last_error(void) { return g_diag_error.c_str(); }

int scoup_diag_set_binsort_segment(int entries_per_segment) {
    if (entries_per_segment < 0 || entries_per_segment > (1 << 24)) {
        g_diag_error = "entries_per_segment out of range";
        return 1;
    }
    scoup::binsort_set_segment_override(entries_per_segment);
    return 0;
}

int scoup_diag_set_raster2_slots(int slots) {
    if (slots != 0 && slots != 4 && slots != 8) {
        g_diag_error = "slots must be 0 (adaptive), 4 or 8";
        return 1;
    }
    scoup::raster2_set_slots_override(slots);
    return 0;
}

int scoup_diag_red_rate(int device, int64_t buffer_bytes, int scattered, int vec4, int64_t reds_per_launch,
                        int launches, double* adds_per_s, double* ms_per_launch) {
    g_diag_error.clear();
    if (!adds_per_s || buffer_bytes < 4096 || reds_per_launch < 1 || launches < 1) {
        g_diag_error = "bad argument";
        return 1;
    }
    int prev = -1;
    cudaGetDevice(&prev);
    cudaSetDevice(device);
    float* buf = nullptr;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    int st = 0;
    auto ck = [&](cudaError_t e, const char* what) {
        if (e != cudaSuccess && st == 0) {
            g_diag_error = std::string(what) + ": " + cudaGetErrorString(e);
            st = 3;
        }
    };
    const uint64_t nfloat = (uint64_t)buffer_bytes / 4;
    ck(cudaMalloc(&buf, (size_t)buffer_bytes), "cudaMalloc");
    if (st == 0) ck(cudaMemset(buf, 0, (size_t)buffer_bytes), "cudaMemset");
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    const int threads = 256, blocks = sms * 8;  // 8 CTAs per SM: 64 warps, full occupancy
    const int64_t instr = vec4 ? (reds_per_launch + 3) / 4 : reds_per_launch;
    const int per_thread = (int)((instr + (int64_t)threads * blocks - 1) / ((int64_t)threads * blocks));
    auto launch = [&](uint32_t salt) {
        if (vec4) {
            if (scattered) red_kernel<true, true><<<blocks, threads>>>(buf, nfloat, per_thread, salt);
            else red_kernel<true, false><<<blocks, threads>>>(buf, nfloat, per_thread, salt);
        } else {
            if (scattered) red_kernel<false, true><<<blocks, threads>>>(buf, nfloat, per_thread, salt);
            else red_kernel<false, false><<<blocks, threads>>>(buf, nfloat, per_thread, salt);
        }
    };
    if (st == 0) {
        ck(cudaEventCreate(&e0), "cudaEventCreate");
        ck(cudaEventCreate(&e1), "cudaEventCreate");
    }
    if (st == 0) {
        launch(0);  // warm-up
        ck(cudaEventRecord(e0), "cudaEventRecord");
        for (int k = 0; k < launches; k++) launch((uint32_t)(k + 1) * 7919u);
        ck(cudaEventRecord(e1), "cudaEventRecord");
        ck(cudaEventSynchronize(e1), "cudaEventSynchronize");
        ck(cudaGetLastError(), "red_kernel");
    }
    if (st == 0) {
        float ms = 0.f;
        ck(cudaEventElapsedTime(&ms, e0, e1), "cudaEventElapsedTime");
        const double adds = (double)per_thread * threads * blocks * (vec4 ? 4.0 : 1.0) * launches;
        *adds_per_s = adds / (ms * 1e-3);
        if (ms_per_launch) *ms_per_launch = ms / launches;
    }
    if (e0) cudaEventDestroy(e0);
    if (e1) cudaEventDestroy(e1);
    if (buf) cudaFree(buf);
    if (prev >= 0) cudaSetDevice(prev);
    return st;
}

}  // extern "C"
