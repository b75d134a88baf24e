// Micro-benchmark of the instruction classes the K-word epilogue is made of
// (DADD, DSETP, 64-bit select, 64-bit integer compare), throughput with many
// independent chains and latency with one dependent chain, on one B200.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/pipe_rates tools/pipe_rates.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kIters = 4096;

template <int OP, int CH>
__global__ void bench(double* out, double seed) {
    double v[CH];
    unsigned long long u[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) {
        v[c] = seed + threadIdx.x * 1e-3 + c;
        u[c] = __double_as_longlong(v[c]);
    }
    const double w = seed * 0.5;
    const unsigned long long uw = __double_as_longlong(w);
    for (int it = 0; it < kIters; ++it) {
#pragma unroll
        for (int c = 0; c < CH; ++c) {
            if (OP == 0) {  // DADD chain
                v[c] = __dadd_rn(v[c], w);
            } else if (OP == 1) {  // DSETP |a| != |b| feeding a select (chain through the select)
                bool p = fabs(v[c]) != fabs(w);
                v[c] = p ? w : v[c];
                asm volatile("" : "+d"(v[c]));
            } else if (OP == 2) {  // 64-bit integer compare feeding a select
                bool p = (u[c] & 0x7fffffffffffffffull) != uw;
                u[c] = p ? uw + it : u[c];
            } else if (OP == 3) {  // DSETP x == 0 (is_zero) feeding a select
                bool p = v[c] == 0.0;
                v[c] = p ? w : __dadd_rn(v[c], 0.0);
            } else if (OP == 4) {  // two_sum (6 dependent-ish DADDs)
                double s = __dadd_rn(v[c], w), bb = __dsub_rn(s, v[c]);
                double e = __dadd_rn(__dsub_rn(v[c], __dsub_rn(s, bb)), __dsub_rn(w, bb));
                v[c] = __dadd_rn(s, e);
            }
        }
    }
    double acc = 0;
#pragma unroll
    for (int c = 0; c < CH; ++c) acc += v[c] + (double)u[c];
    if (acc == 1.2345) out[threadIdx.x] = acc;
}

template <int OP, int CH>
void run(const char* name, int warps_per_sm, int ops_per_iter) {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* out;
    cudaMalloc(&out, 4096 * 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    bench<OP, CH><<<sms, warps_per_sm * 32>>>(out, 1.5);
    cudaEventRecord(e0);
    bench<OP, CH><<<sms, warps_per_sm * 32>>>(out, 1.5);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    int clk;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const double cycles = ms * 1e-3 * clk * 1e3;
    const double warp_instr = (double)warps_per_sm * kIters * CH * ops_per_iter;  // per SM
    printf("%-34s warps/SM %2d chains %d: %.3f warp-ops/clk/SM, %.1f clk per dependent op\n", name,
           warps_per_sm, CH, warp_instr / cycles, cycles / ((double)kIters * ops_per_iter));
    cudaFree(out);
}

int main() {
    run<0, 8>("DADD throughput", 32, 1);
    run<0, 1>("DADD latency", 4, 1);
    run<1, 8>("DSETP|abs| + sel throughput", 32, 1);
    run<1, 1>("DSETP|abs| + sel latency", 4, 1);
    run<3, 8>("DSETP==0 + sel + DADD throughput", 32, 1);
    run<2, 8>("u64 cmp + sel throughput", 32, 1);
    run<2, 1>("u64 cmp + sel latency", 4, 1);
    run<4, 8>("two_sum throughput (6 DADD)", 32, 1);
    run<4, 1>("two_sum+add latency (7 DADD)", 4, 1);
    return 0;
}
