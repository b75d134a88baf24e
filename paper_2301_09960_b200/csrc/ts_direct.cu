// ts_direct.cu -- K5: direct triple-single GEMM, the comparator of BASELINE
// config 4 ("TS Ozaki GEMM n=8192 vs direct TS GEMM kernel").
//
// The reference has no TS code.  The paper's GPU direct TS GEMM
// accumulates triple-single dot products with TwoProd /
// TwoSum in binary32; its exact operation sequence is defined in
// oracle/ozk_oracle.c (ozk_oracle_ts_fma) and replayed here bit for bit:
// every output element is accumulated in strictly ascending k, one TS
// multiply-accumulate per term, with explicit round-to-nearest intrinsics (no
// contraction except the TwoProd error FMAs).
//
// B200 mapping: FP32 SIMT (the work is ~65 dependent binary32 ops per term,
// not a contraction a tensor core can do).  64x64 C tile per 256-thread CTA,
// 4x4 outputs per thread (12 accumulator words), 16-deep k tiles staged in
// shared memory as [k][word][row] so each thread reads its 4 rows / 4 columns
// of one word with a single LDS.128; the next k tile is prefetched into
// registers while the current one is consumed.
#include <cuda_runtime.h>

#include "ozk_internal.cuh"

namespace ozk {
namespace {

constexpr int TM = 64, TN = 64, TK = 16, kThreads = 256;

__device__ __forceinline__ void two_sum_f(float a, float b, float& s, float& e) {
    const float ss = __fadd_rn(a, b);
    const float bb = __fsub_rn(ss, a);
    e = __fadd_rn(__fsub_rn(a, __fsub_rn(ss, bb)), __fsub_rn(b, bb));
    s = ss;
}

// ozk_oracle_ts_fma: s += a * b in triple-single
__device__ __forceinline__ void ts_fma(float& s0, float& s1, float& s2, float a0, float a1,
                                       float a2, float b0, float b1, float b2) {
    const float p00 = __fmul_rn(a0, b0), e00 = __fmaf_rn(a0, b0, -p00);
    const float p01 = __fmul_rn(a0, b1), e01 = __fmaf_rn(a0, b1, -p01);
    const float p10 = __fmul_rn(a1, b0), e10 = __fmaf_rn(a1, b0, -p10);
    const float t2 = __fadd_rn(__fadd_rn(__fadd_rn(__fmul_rn(a0, b2), __fmul_rn(a1, b1)),
                                         __fmul_rn(a2, b0)),
                               __fadd_rn(e01, e10));
    float r0, q, r1, r2, r3, r4;
    two_sum_f(s0, p00, s0, r0);
    two_sum_f(p01, p10, q, r1);
    two_sum_f(q, e00, q, r2);
    two_sum_f(s1, q, s1, r3);
    two_sum_f(s1, r0, s1, r4);
    s2 = __fadd_rn(__fadd_rn(__fadd_rn(__fadd_rn(s2, t2), r1), r2), __fadd_rn(r3, r4));
    two_sum_f(s1, s2, s1, s2);
    two_sum_f(s0, s1, s0, s1);
    two_sum_f(s1, s2, s1, s2);
}

__global__ void __launch_bounds__(kThreads)
ts_direct_kernel(const float* __restrict__ A, const float* __restrict__ B, float* __restrict__ C,
                 int m, int l, int n) {
    __shared__ __align__(16) float As[2][TK][3][TM];
    __shared__ __align__(16) float Bs[2][TK][3][TN];
    const int tid = threadIdx.x;
    const int tx = tid & 15, ty = tid >> 4;
    const int row0 = blockIdx.y * TM, col0 = blockIdx.x * TN;

    // global -> register staging: A thread loads row (tid/4), k range (tid%4)*4..+3;
    // B thread loads k (tid/16), columns (tid%16)*4..+3; 12 words each.
    const int a_r = tid >> 2, a_k = (tid & 3) * 4;
    const int b_k = tid >> 4, b_c = (tid & 15) * 4;
    float ra[12], rb[12];
    auto load = [&](int k0) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int gr = row0 + a_r, gk = k0 + a_k + q;
            const bool ok = gr < m && gk < l;
            const float* p = A + ((size_t)gr * l + gk) * 3;
#pragma unroll
            for (int w = 0; w < 3; ++w) ra[q * 3 + w] = ok ? p[w] : 0.0f;
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int gk = k0 + b_k, gc = col0 + b_c + q;
            const bool ok = gk < l && gc < n;
            const float* p = B + ((size_t)gk * n + gc) * 3;
#pragma unroll
            for (int w = 0; w < 3; ++w) rb[q * 3 + w] = ok ? p[w] : 0.0f;
        }
    };
    auto store = [&](int buf) {
#pragma unroll
        for (int q = 0; q < 4; ++q)
#pragma unroll
            for (int w = 0; w < 3; ++w) As[buf][a_k + q][w][a_r] = ra[q * 3 + w];
#pragma unroll
        for (int q = 0; q < 4; ++q)
#pragma unroll
            for (int w = 0; w < 3; ++w) Bs[buf][b_k][w][b_c + q] = rb[q * 3 + w];
    };

    float s[4][4][3];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) s[i][j][0] = s[i][j][1] = s[i][j][2] = 0.0f;

    const int ntiles = (l + TK - 1) / TK;
    load(0);
    store(0);
    __syncthreads();
    for (int t = 0; t < ntiles; ++t) {
        const int buf = t & 1;
        if (t + 1 < ntiles) load((t + 1) * TK);
        const int kmax = min(TK, l - t * TK);  // padded k terms are never added
        for (int k = 0; k < kmax; ++k) {
            float a[3][4], b[3][4];
#pragma unroll
            for (int w = 0; w < 3; ++w) {
                const float4 av = *reinterpret_cast<const float4*>(&As[buf][k][w][ty * 4]);
                const float4 bv = *reinterpret_cast<const float4*>(&Bs[buf][k][w][tx * 4]);
                a[w][0] = av.x; a[w][1] = av.y; a[w][2] = av.z; a[w][3] = av.w;
                b[w][0] = bv.x; b[w][1] = bv.y; b[w][2] = bv.z; b[w][3] = bv.w;
            }
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    ts_fma(s[i][j][0], s[i][j][1], s[i][j][2], a[0][i], a[1][i], a[2][i],
                           b[0][j], b[1][j], b[2][j]);
        }
        if (t + 1 < ntiles) {
            store(buf ^ 1);
            __syncthreads();
        }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int gr = row0 + ty * 4 + i;
        if (gr >= m) continue;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int gc = col0 + tx * 4 + j;
            if (gc >= n) continue;
            float* p = C + ((size_t)gr * n + gc) * 3;
            p[0] = s[i][j][0];
            p[1] = s[i][j][1];
            p[2] = s[i][j][2];
        }
    }
}

} // namespace

cudaError_t launch_ts_direct(const float* a, const float* b, float* c, size_t m, size_t l,
                             size_t n, cudaStream_t st) {
    if (m == 0 || n == 0) return cudaSuccess;
    dim3 grid((unsigned)((n + TN - 1) / TN), (unsigned)((m + TM - 1) / TM));
    ts_direct_kernel<<<grid, kThreads, 0, st>>>(a, b, c, (int)m, (int)l, (int)n);
    return cudaGetLastError();
}

} // namespace ozk
