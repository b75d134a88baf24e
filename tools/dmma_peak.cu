// FP64 tensor (DMMA) and scalar DFMA peak microbenchmark for sm_100a.
//
// The driver's MEASURED_PEAKS.json carries HBM and bf16 peaks only; the Ozaki
// slice GEMMs are bounded by the FP64 tensor pipe, so the roofline denominator
// for them is measured here: register-resident mma.sync.m8n8k4.f64 chains,
// one launch over all SMs, timed with CUDA events.
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dmma_peak dmma_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
    std::printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); return 1; } } while (0)

template <int CHAINS>
__global__ void dmma_loop(double* out, int iters, double seed) {
    double a = seed + threadIdx.x * 1e-3, b = seed * 0.5 + 1.0;
    double c0[CHAINS], c1[CHAINS];
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) { c0[i] = 0.0; c1[i] = 0.0; }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < CHAINS; ++i) {
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                         : "+d"(c0[i]), "+d"(c1[i]) : "d"(a), "d"(b));
        }
    }
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) s += c0[i] + c1[i];
    if (s == 12345.678) out[0] = s;
}

template <int CHAINS>
__global__ void dfma_loop(double* out, int iters, double seed) {
    double a = seed + threadIdx.x * 1e-3, b = 0.999999;
    double c[CHAINS];
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) c[i] = i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < CHAINS; ++i) c[i] = fma(c[i], b, a);
    }
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) s += c[i];
    if (s == 12345.678) out[0] = s;
}

int main() {
    cudaDeviceProp p;
    CK(cudaGetDeviceProperties(&p, 0));
    int sms = p.multiProcessorCount;
    int clk_khz = 0;
    cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
    std::printf("{\"device\": \"%s\", \"sms\": %d, \"clock_khz\": %d}\n", p.name, sms, clk_khz);
    double* out;
    CK(cudaMalloc(&out, 8));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 20000;
    for (int warps : {4, 8, 16}) {
        dim3 grid(sms * 1), block(32 * warps);
        dmma_loop<8><<<grid, block>>>(out, 100, 1.0);
        CK(cudaDeviceSynchronize());
        float best = 1e30f;
        for (int r = 0; r < 5; ++r) {
            cudaEventRecord(e0);
            dmma_loop<8><<<grid, block>>>(out, iters, 1.0);
            cudaEventRecord(e1);
            CK(cudaEventSynchronize(e1));
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (ms < best) best = ms;
        }
        double flops = 2.0 * 256.0 * 8 * double(iters) * warps * sms;
        std::printf("{\"kind\": \"dmma_m8n8k4\", \"warps_per_sm\": %d, \"ms\": %.3f, \"tflops\": %.3f}\n",
                    warps, best, flops / best / 1e9);
    }
    for (int warps : {8, 16, 32}) {
        dim3 grid(sms), block(32 * warps);
        dfma_loop<8><<<grid, block>>>(out, 100, 1.0);
        CK(cudaDeviceSynchronize());
        float best = 1e30f;
        for (int r = 0; r < 5; ++r) {
            cudaEventRecord(e0);
            dfma_loop<8><<<grid, block>>>(out, iters, 1.0);
            cudaEventRecord(e1);
            CK(cudaEventSynchronize(e1));
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (ms < best) best = ms;
        }
        double flops = 2.0 * 8 * double(iters) * 32 * warps * sms;
        std::printf("{\"kind\": \"dfma\", \"warps_per_sm\": %d, \"ms\": %.3f, \"tflops\": %.3f}\n",
                    warps, best, flops / best / 1e9);
    }
    return 0;
}
