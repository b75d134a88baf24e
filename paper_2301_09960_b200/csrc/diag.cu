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

// ---- tcgen05 kind::i8 ceiling (roofline denominator of the INT8 engine) -----
// One CTA per SM issues back-to-back tcgen05.mma.kind::i8 (M=128, N=256, K=32)
// from shared memory into TMEM: no data movement, so this is the dense INT8
// tensor ceiling reachable from a single-CTA (cta_group::1) issuer.
namespace {

__device__ __forceinline__ uint64_t probe_desc(uint32_t saddr) {
    return (uint64_t)((saddr >> 4) & 0x3fff) | ((uint64_t)1 << 16) |
           ((uint64_t)(1024 >> 4) << 32) | ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}

__global__ void __launch_bounds__(128) i8_probe_kernel(int iters, int* sink) {
    extern __shared__ __align__(1024) uint8_t sm[];
    uint8_t* base = (uint8_t*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
    __shared__ uint64_t bar;
    __shared__ uint32_t tmem_slot;
    const int warp = threadIdx.x / 32;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(
            (uint32_t)__cvta_generic_to_shared(&tmem_slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = tmem_slot;
    if (threadIdx.x == 0) {
        const uint32_t sa = (uint32_t)__cvta_generic_to_shared(base);
        const uint32_t sb = sa + 128 * 128;
        constexpr uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((256u >> 3) << 17) |
                                   ((128u >> 4) << 24);
        for (int it = 0; it < iters; ++it)
#pragma unroll
            for (int k = 0; k < 4; ++k)
                asm volatile(
                    "{ .reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p; }" ::"r"(tmem),
                    "l"(probe_desc(sa + k * 32)), "l"(probe_desc(sb + k * 32)), "r"(idesc), "r"(it | k));
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                         (uint32_t)__cvta_generic_to_shared(&bar))
                     : "memory");
        uint32_t ok = 0;
        while (!ok)
            asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0,1,0,p; }"
                         : "=r"(ok)
                         : "r"((uint32_t)__cvta_generic_to_shared(&bar))
                         : "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
    if (iters < 0) sink[0] = 1;
}

}  // namespace

extern "C" double ozk_probe_i8_tops(int iters, void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int smem = 128 * 128 + 256 * 128 + 1024;
    if (cudaFuncSetAttribute(i8_probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) !=
        cudaSuccess)
        return -1.0;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    i8_probe_kernel<<<sms, 128, smem, st>>>(64, nullptr);
    float best = 1e30f;
    for (int r = 0; r < 3; ++r) {
        cudaEventRecord(e0, st);
        i8_probe_kernel<<<sms, 128, smem, st>>>(iters, nullptr);
        cudaEventRecord(e1, st);
        cudaEventSynchronize(e1);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    if (cudaStreamSynchronize(st) != cudaSuccess) return -1.0;
    const double ops = 2.0 * 128.0 * 256.0 * 32.0 * 4.0 * (double)iters * sms;
    return ops / (best * 1e-3) / 1e12;
}
