// Does tcgen05 MMA traffic slow the SM's FP64 pipe?  One CTA per SM: warp 0
// (optionally) streams tcgen05.mma kind::i8 M=128 N=192 K=32 from shared memory
// into TMEM while warps 1..W run independent dependent-DADD chains (the
// K-word epilogue's instruction class); the DADD warps report their rate.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/contention_probe tools/contention_probe.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kChains = 4;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ uint64_t desc(uint32_t a) {
    return (uint64_t)((a >> 4) & 0x3fff) | (1ull << 16) | ((uint64_t)(1024 >> 4) << 32) |
           (1ull << 46) | (2ull << 61);
}

template <int MN>
__global__ void __launch_bounds__(544, 1) probe(int mma_on, int mma_iters, int dadd_iters,
                                                unsigned long long* out, double seed) {
    extern __shared__ __align__(1024) uint8_t sm_raw[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint32_t tslot;
    __shared__ uint64_t bar;
    const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(&tslot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = tslot;
    if (warp == 0) {
        if (mma_on && lane == 0) {
            const uint32_t a = smem_u32(sm), b = a + 16384;
            const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(MN >> 3) << 17) | ((128u >> 4) << 24);
            for (int i = 0; i < mma_iters; ++i)
                asm volatile("{ .reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p; }"
                             ::"r"(tmem), "l"(desc(a + (i & 3) * 32)), "l"(desc(b + (i & 3) * 32)), "r"(idesc), "r"(i));
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)) : "memory");
            uint32_t ok = 0;
            while (!ok)
                asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0,1,0,p; }"
                             : "=r"(ok) : "r"(smem_u32(&bar)) : "memory");
        }
    } else {
        double v[kChains];
#pragma unroll
        for (int c = 0; c < kChains; ++c) v[c] = seed + threadIdx.x * 1e-3 + c;
        const double w = seed * 0.5;
        const unsigned long long t0 = clock64();
        for (int it = 0; it < dadd_iters; ++it) {
#pragma unroll
            for (int c = 0; c < kChains; ++c) v[c] = __dadd_rn(v[c], w);
        }
        const unsigned long long t1 = clock64();
        double acc = 0;
#pragma unroll
        for (int c = 0; c < kChains; ++c) acc += v[c];
        if (lane == 0) out[blockIdx.x * 32 + warp] = t1 - t0;
        if (acc == 1.25) out[0] = 0;
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
}

template <int MN>
void run(int sms, unsigned long long* out, int smem, int dadd_iters, int warps, int on);

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    unsigned long long* out;
    cudaMalloc(&out, sizeof(unsigned long long) * sms * 32);
    const int smem = 16384 + 32768 + 2048;  // A 128x128 B, B up to 256x128 B (+ align)
    const int dadd_iters = 200000;
    run<192>(sms, out, smem, dadd_iters, 16, 0);
    for (int on = 1; on < 2; ++on)
        for (int mn : {64, 128, 192, 256}) {
            if (mn == 64) run<64>(sms, out, smem, dadd_iters, 16, on);
            if (mn == 128) run<128>(sms, out, smem, dadd_iters, 16, on);
            if (mn == 192) run<192>(sms, out, smem, dadd_iters, 16, on);
            if (mn == 256) run<256>(sms, out, smem, dadd_iters, 16, on);
        }
    return 0;
}

template <int MN>
void run(int sms, unsigned long long* out, int smem, int dadd_iters, int warps, int on) {
    cudaFuncSetAttribute(probe<MN>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    {
        {
            cudaEvent_t e0, e1;
            cudaEventCreate(&e0);
            cudaEventCreate(&e1);
            probe<MN><<<sms, 32 * (1 + warps), smem>>>(on, 1, 1000, out, 1.5);  // warm
            cudaEventRecord(e0);
            // MMA count scaled so the MMA stream outlasts the DADD loop
            probe<MN><<<sms, 32 * (1 + warps), smem>>>(on, 60000 * 256 / MN, dadd_iters, out, 1.5);
            cudaEventRecord(e1);
            cudaError_t err = cudaEventSynchronize(e1);
            float ms = 0;
            cudaEventElapsedTime(&ms, e0, e1);
            unsigned long long h[32];
            cudaMemcpy(h, out, sizeof(h), cudaMemcpyDeviceToHost);
            double cyc = 0;
            for (int w = 1; w <= warps; ++w) cyc += (double)h[w];
            cyc /= warps;
            const double per = cyc / dadd_iters;  // cycles per iteration (kChains DADDs per warp)
            printf("dadd warps %2d mma %s N=%3d: %.2f clk per chain step (%d chains/warp) -> %.3f DADD warp-ops/clk/SM; kernel %.2f ms %s\n",
                   warps, on ? "ON " : "off", MN, per, kChains, warps * kChains / per, ms,
                   err == cudaSuccess ? "" : cudaGetErrorString(err));
        }
    }
}
