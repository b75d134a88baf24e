// lu.cu -- the blocked-LU trailing update's K-word subtraction as a separate
// pass, A22(i, j) -= update(i, j) (proj/include/mpmat/lu.hpp:121-124).  The
// slice GEMMs fuse it into their last pair's epilogue (LuTarget in api.cu);
// this pass serves the one case without a last pair (every pair pruned:
// A22 -= 0 still goes through the reference's subtraction).
// The subtraction is MultiFloat<K>::operator-=(MultiFloat<K>)
// (multifloat.hpp:300,201: x + (-y)), replayed by kw_add_kw (kword.cuh).
// Memory-bound elementwise pass: 3*K*8 bytes per element.
#include "kword.cuh"
#include "ozk_internal.cuh"

namespace ozk {
namespace {

template <int K>
__global__ void kw_sub_inplace_kernel(double* __restrict__ a, size_t lda,
                                      const double* __restrict__ c, size_t rows, size_t cols) {
    const size_t total = rows * cols;
    for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < total;
         e += (size_t)gridDim.x * blockDim.x) {
        const size_t i = e / cols, j = e - i * cols;
        double* ap = a + (i * lda + j) * K;
        const double* cp = c + e * K;
        double x[K], y[K], ny[K];
#pragma unroll
        for (int k = 0; k < K; ++k) {
            x[k] = ap[k];
            y[k] = cp[k];
        }
        kw_neg<K>(y, ny);
        kw_add_kw<K>(x, ny);
#pragma unroll
        for (int k = 0; k < K; ++k) ap[k] = x[k];
    }
}

} // namespace

cudaError_t launch_kw_sub_inplace(int K, double* a, size_t lda, const double* c, size_t rows,
                                  size_t cols, cudaStream_t st) {
    if (rows == 0 || cols == 0) return cudaSuccess;
    const int threads = 256;
    size_t blocks = (rows * cols + threads - 1) / threads;
    if (blocks > 148 * 32) blocks = 148 * 32;
    switch (K) {
    case 2: kw_sub_inplace_kernel<2><<<(unsigned)blocks, threads, 0, st>>>(a, lda, c, rows, cols); break;
    case 3: kw_sub_inplace_kernel<3><<<(unsigned)blocks, threads, 0, st>>>(a, lda, c, rows, cols); break;
    case 4: kw_sub_inplace_kernel<4><<<(unsigned)blocks, threads, 0, st>>>(a, lda, c, rows, cols); break;
    default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

} // namespace ozk
