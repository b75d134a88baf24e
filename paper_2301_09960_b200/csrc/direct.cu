// direct.cu -- the direct K-word GEMM: the reference's
// gemm_simple<MultiFloat<K>> (proj/include/mpmat/gemm.hpp:15-31) on the GPU,
// bit for bit: every C element is  c = 0;  for k = 0..l-1:  c = c + a(i,k) * b(k,j)
// with the reference's MultiFloat<K> multiply (multifloat.hpp:218-239,
// kw_mul_kw) and add (:184-199, kw_add_kw), in that fixed k order.
//
// It is the comparator the paper measures the Ozaki scheme against, not a hot
// path: one thread per C element (its k loop is inherently sequential), 16x16
// elements per CTA, A/B K-word tiles of 16-deep k staged in shared memory so a
// loaded word serves 16 threads.  The work is the long-precision arithmetic
// (a few hundred FP64 ops per multiply-add), so the roofline is the FP64 pipe.
#include "kword.cuh"
#include "ozk_internal.cuh"

namespace ozk {
namespace {

constexpr int kTile = 16;

template <int K>
__global__ void __launch_bounds__(kTile * kTile)
direct_gemm_kernel(const double* __restrict__ a, const double* __restrict__ b,
                   double* __restrict__ c, size_t m, size_t l, size_t n) {
    __shared__ double sa[kTile][kTile][K];      // [row][k]
    __shared__ double sb[kTile][kTile][K + 1];  // [k][col], padded
    const int tx = threadIdx.x % kTile, ty = threadIdx.x / kTile;
    const size_t i = (size_t)blockIdx.y * kTile + ty;
    const size_t j = (size_t)blockIdx.x * kTile + tx;
    double acc[K];
#pragma unroll
    for (int q = 0; q < K; ++q) acc[q] = 0.0;
    for (size_t k0 = 0; k0 < l; k0 += kTile) {
        // tile loads (zero outside the matrix: never used, k is bounded below)
        {
            const size_t ar = (size_t)blockIdx.y * kTile + ty, ak = k0 + tx;
#pragma unroll
            for (int q = 0; q < K; ++q)
                sa[ty][tx][q] = (ar < m && ak < l) ? a[(ar * l + ak) * K + q] : 0.0;
            const size_t bk = k0 + ty, bc = (size_t)blockIdx.x * kTile + tx;
#pragma unroll
            for (int q = 0; q < K; ++q)
                sb[ty][tx][q] = (bk < l && bc < n) ? b[(bk * n + bc) * K + q] : 0.0;
        }
        __syncthreads();
        const int kk_end = (int)((l - k0) < (size_t)kTile ? (l - k0) : (size_t)kTile);
        if (i < m && j < n) {
            for (int kk = 0; kk < kk_end; ++kk) {
                double x[K], y[K], p[K];
#pragma unroll
                for (int q = 0; q < K; ++q) {
                    x[q] = sa[ty][kk][q];
                    y[q] = sb[kk][tx][q];
                }
                kw_mul_kw<K>(x, y, p);
                kw_add_kw<K>(acc, p);  // c(i,j) += a(i,k) * b(k,j)  (gemm.hpp:29)
            }
        }
        __syncthreads();
    }
    if (i < m && j < n) {
#pragma unroll
        for (int q = 0; q < K; ++q) c[(i * n + j) * K + q] = acc[q];
    }
}

}  // namespace

cudaError_t launch_direct_gemm(int K, const double* a, const double* b, double* c, size_t m,
                               size_t l, size_t n, cudaStream_t st) {
    const dim3 grid((unsigned)((n + kTile - 1) / kTile), (unsigned)((m + kTile - 1) / kTile));
    switch (K) {
    case 2: direct_gemm_kernel<2><<<grid, kTile * kTile, 0, st>>>(a, b, c, m, l, n); break;
    case 3: direct_gemm_kernel<3><<<grid, kTile * kTile, 0, st>>>(a, b, c, m, l, n); break;
    case 4: direct_gemm_kernel<4><<<grid, kTile * kTile, 0, st>>>(a, b, c, m, l, n); break;
    default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

}  // namespace ozk
