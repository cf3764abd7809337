// CUDA-core 32-bit add throughput on this device: the roofline denominator of the
// dedispersion kernel, which is ALU-bound (~460 channel-adds per algorithmic byte,
// SURVEY.md section 8d), not HBM- or tensor-bound.
//
// Three dependent-but-wide add patterns (16 accumulators, ILP 8, not foldable):
//   0: integer IADD only (ALU pipe), 1: FADD only (FMA pipe), 2: both interleaved.
// The reported peak is the best of the three in lane-adds per second.
#include "pgb_internal.h"

namespace pgb {
namespace {

template <int MODE>
__global__ void __launch_bounds__(256) add_peak_kernel(uint32_t iters, uint32_t* sink) {
    uint32_t a[16];
    float f[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) {
        a[k] = threadIdx.x * 16u + k;
        f[k] = 1e-30f * (float)(k + 1);
    }
    for (uint32_t it = 0; it < iters; ++it) {
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            if (MODE == 0 || (MODE == 2 && (k & 1) == 0)) a[k] = a[k] + a[(k + 8) & 15];
            if (MODE == 1 || (MODE == 2 && (k & 1) == 1)) f[k] = __fadd_rn(f[k], f[(k + 8) & 15]);
        }
    }
    uint32_t r = 0;
#pragma unroll
    for (int k = 0; k < 16; ++k) r ^= a[k] ^ __float_as_uint(f[k]);
    if (r == 0x9e3779b9u) sink[0] = r;  // practically never; keeps the adds live
}

}  // namespace
}  // namespace pgb

using namespace pgb;

extern "C" pgb_status pgb_microbench_add_peak(int device, double* adds_per_s, double* per_mode) {
    try {
        PGB_CUDA(cudaSetDevice(device));
        int sms = 0;
        PGB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
        uint32_t* sink = nullptr;
        PGB_CUDA(cudaMalloc(&sink, 4));
        cudaEvent_t e0, e1;
        PGB_CUDA(cudaEventCreate(&e0));
        PGB_CUDA(cudaEventCreate(&e1));
        const uint32_t iters = 8192;
        const unsigned blocks = (unsigned)sms * 8, threads = 256;
        double best = 0.0;
        for (int mode = 0; mode < 3; ++mode) {
            float ms = 0.f, best_ms = 1e30f;
            for (int rep = 0; rep < 4; ++rep) {
                PGB_CUDA(cudaEventRecord(e0));
                if (mode == 0) add_peak_kernel<0><<<blocks, threads>>>(iters, sink);
                else if (mode == 1) add_peak_kernel<1><<<blocks, threads>>>(iters, sink);
                else add_peak_kernel<2><<<blocks, threads>>>(iters, sink);
                PGB_CUDA(cudaEventRecord(e1));
                PGB_CUDA(cudaEventSynchronize(e1));
                PGB_CUDA(cudaEventElapsedTime(&ms, e0, e1));
                if (rep > 0) best_ms = std::min(best_ms, ms);  // first launch is warm-up
            }
            const double adds = (double)blocks * threads * iters * 16.0;
            const double rate = adds / (best_ms * 1e-3);
            if (per_mode) per_mode[mode] = rate;
            best = std::max(best, rate);
        }
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        cudaFree(sink);
        if (adds_per_s) *adds_per_s = best;
        return PGB_OK;
    } catch (const Error& e) {
        return e.code;
    }
}
