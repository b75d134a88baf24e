// accumulate.cu -- the reference's stand-alone accumulation phase (ozaki.hpp:
// 235-244): per element, acc = 0; for p in pair order: acc += C_p, with
// MultiFloat<K> + double (kword.cuh kw_add, the reference operation sequence).
//
// The fused engines never need it (the same adds run in the slice-GEMM
// epilogue).  It serves callers that bring their own GemmBackend
// (mpmat::gpu::ozaki_gemm with a non-B200 backend, include/mpmat_gpu.hpp): the
// split runs on the GPU, the caller's backend forms every C_ab, and this pass
// sums them.  HBM-bound: nproducts * 8 + K * word bytes per element.
#include "kword.cuh"
#include "ozk_internal.cuh"

namespace ozk {
namespace {

template <int K, typename W>
__global__ void accumulate_kernel(const double* __restrict__ prods, int np, size_t count,
                                  W* __restrict__ c) {
    for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < count;
         e += (size_t)gridDim.x * blockDim.x) {
        W acc[K];
#pragma unroll
        for (int k = 0; k < K; ++k) acc[k] = W(0);
        for (int p = 0; p < np; ++p)
            kw_add<K, W, true, true>(acc, (W)prods[(size_t)p * count + e]);
#pragma unroll
        for (int k = 0; k < K; ++k) c[e * K + k] = acc[k];
    }
}

}  // namespace

cudaError_t launch_accumulate_products(int K, int word_bytes, const double* prods, int np,
                                       size_t count, void* c, cudaStream_t st) {
    if (count == 0) return cudaSuccess;
    const int threads = 256;
    size_t blocks = (count + threads - 1) / threads;
    if (blocks > 148 * 32) blocks = 148 * 32;
    const unsigned g = (unsigned)blocks;
    if (word_bytes == 4) {
        if (K != 3) return cudaErrorInvalidValue;
        accumulate_kernel<3, float><<<g, threads, 0, st>>>(prods, np, count, static_cast<float*>(c));
        return cudaGetLastError();
    }
    switch (K) {
    case 2: accumulate_kernel<2, double><<<g, threads, 0, st>>>(prods, np, count, static_cast<double*>(c)); break;
    case 3: accumulate_kernel<3, double><<<g, threads, 0, st>>>(prods, np, count, static_cast<double*>(c)); break;
    case 4: accumulate_kernel<4, double><<<g, threads, 0, st>>>(prods, np, count, static_cast<double*>(c)); break;
    default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

}  // namespace ozk
