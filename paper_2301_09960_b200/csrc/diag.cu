// diag.cu -- in-run FP64 tensor-pipe peak probe (the roofline denominator).
//
// MEASURED_PEAKS.json (driver-written) carries HBM and bf16 peaks only; the
// Ozaki slice GEMMs are bounded by the FP64 DMMA pipe, so bench.py measures
// that pipe's ceiling in the same process, right before its timed region:
// register-resident, dependency-free chains of mma.sync.m8n8k4.f64 (SASS
// DMMA.8x8x4) on every SM, no memory traffic.  Same method as
// tools/dmma_peak.cu (37.1 TFLOP/s measured on B200 at 1965 MHz).
#include <cuda_runtime.h>

#include "../../include/ozk.h"

namespace {

__global__ void __launch_bounds__(256) dmma_probe_kernel(double* out, int iters, double seed) {
    double a = seed + threadIdx.x * 1e-3, b = seed * 0.5 + 1.0;
    double c0[8], c1[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) c0[i] = c1[i] = 0.0;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                         : "+d"(c0[i]), "+d"(c1[i])
                         : "d"(a), "d"(b));
    }
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += c0[i] + c1[i];
    if (s == 12345.678) out[0] = s;
}

}  // namespace

extern "C" double ozk_probe_dmma_tflops(int iters, void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    double* out = nullptr;
    if (cudaMallocAsync(&out, 8, st) != cudaSuccess) return -1.0;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    dmma_probe_kernel<<<sms, 256, 0, st>>>(out, 64, 1.0);  // warm-up
    float best = 1e30f;
    for (int r = 0; r < 3; ++r) {
        cudaEventRecord(e0, st);
        dmma_probe_kernel<<<sms, 256, 0, st>>>(out, iters, 1.0);
        cudaEventRecord(e1, st);
        cudaEventSynchronize(e1);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFreeAsync(out, st);
    if (cudaStreamSynchronize(st) != cudaSuccess) return -1.0;
    const double flops = 2.0 * 256.0 * 8.0 * (double)iters * 8.0 /*warps*/ * sms;
    return flops / (best * 1e-3) / 1e12;
}
