// split.cu -- K1: the Ozaki split (error-free extraction of FP64 slices) and
// the K-word transpose that turns the B-side (per-column) split into a per-row
// one with k-contiguous output slices.
//
// Reference: split_matrix<K> (proj/include/mpmat/ozaki.hpp:74-147) with
// exponent_ceil_log2 (:36-40), shift_extract (:53-56), leading_image and the
// per-row max (dense_matrix.hpp:72-96) and MultiFloat<K>::operator-=(double)
// (multifloat.hpp:304 -> :290-300).
//
// Layout: one CTA owns one row (A side) / one column (B side, after the
// transpose) and runs all D extraction passes on it, so the D dependent
// row-max reductions are CTA-local (warp shuffles + one smem hop) and never
// touch the grid.  The K-word residual is swept once per pass through the
// `work` buffer; a row is at most l*K*8 bytes (256 KiB for QD at l=8192), and
// 512-thread CTAs keep ~2 resident rows per SM, so the per-pass re-reads mostly
// stay in L2.  Slices are written k-contiguous with a 16-byte padded
// leading dimension, which is the operand layout the DMMA GEMM's TMA loads.
#include "kword.cuh"
#include "ozk_internal.cuh"

namespace ozk {
namespace {

#ifndef OZK_SPLIT_THREADS
// 512-thread CTAs, two per SM (50-64 registers; the ~300 resident rows'
// residuals, 57 MB at TD l = 8192, fit L2): DD / TD / QD split 5.9 / 18.4 /
// 29.5 ms; 256, 384, 768 and 1024 threads measured slower (TD 19.1-26.8 ms)
#define OZK_SPLIT_THREADS 512
#endif
constexpr int kSplitThreads = OZK_SPLIT_THREADS;

__device__ __forceinline__ int ceil_log2(double x) {
    int e = ilogb(x);
    return scalbn(1.0, e) == x ? e : e + 1;
}
__device__ __forceinline__ int ceil_log2(float x) {
    int e = ilogbf(x);
    return scalbnf(1.0f, e) == x ? e : e + 1;
}
__device__ __forceinline__ double pow2(double, int e) { return scalbn(1.0, e); }
__device__ __forceinline__ float pow2(float, int e) { return scalbnf(1.0f, e); }

// "entries too large to shift" guard: ozaki.hpp:109 keeps e + sigma <= 1020
// (3 binades below binary64's 1023); TS keeps the same margin below 127.
template <typename T> struct ShiftGuard;
template <> struct ShiftGuard<double> { static constexpr int max_exp = 1020; static constexpr int S = 53; };
template <> struct ShiftGuard<float> { static constexpr int max_exp = 124; static constexpr int S = 24; };

// Block-wide max of a non-negative double; every thread gets the result.
__device__ __forceinline__ double block_max(double v, double* red) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, off));
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) red[warp] = v;
    __syncthreads();
    if (warp == 0) {
        v = lane < (int)(blockDim.x >> 5) ? red[lane] : 0.0;
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, off));
        if (lane == 0) red[32] = v;
    }
    __syncthreads();
    v = red[32];
    __syncthreads();
    return v;
}

template <int K, typename T>
__device__ __forceinline__ void load_kw(const T* p, T* c) {
    if constexpr (K == 2 && sizeof(T) == 8) {
        double2 v = *reinterpret_cast<const double2*>(p);
        c[0] = v.x;
        c[1] = v.y;
    } else if constexpr (K == 4 && sizeof(T) == 8) {
        double2 v0 = reinterpret_cast<const double2*>(p)[0];
        double2 v1 = reinterpret_cast<const double2*>(p)[1];
        c[0] = v0.x;
        c[1] = v0.y;
        c[2] = v1.x;
        c[3] = v1.y;
    } else {
#pragma unroll
        for (int k = 0; k < K; ++k) c[k] = p[k];
    }
}

template <int K, typename T>
__device__ __forceinline__ void store_kw(T* p, const T* c) {
    if constexpr (K == 2 && sizeof(T) == 8) {
        *reinterpret_cast<double2*>(p) = make_double2(c[0], c[1]);
    } else if constexpr (K == 4 && sizeof(T) == 8) {
        reinterpret_cast<double2*>(p)[0] = make_double2(c[0], c[1]);
        reinterpret_cast<double2*>(p)[1] = make_double2(c[2], c[3]);
    } else {
#pragma unroll
        for (int k = 0; k < K; ++k) p[k] = c[k];
    }
}

// T is the word type of the K-word input/residual (double: DD/TD/QD, float:
// TS); slices are always written as binary64 (a TS slice is a binary32 value,
// exactly representable), which is the DMMA GEMM's operand type.
//
// NT threads per CTA (one row per CTA).  SM: the K-word residual row lives in
// shared memory across the D passes (rows up to ~220 KB: TD/DD/TS at l = 8192,
// not QD) -- one 1024-thread CTA per SM, and the per-pass residual sweeps
// become shared-memory traffic instead of L2/DRAM round trips (the global
// variant, two 512-thread CTAs per SM, wrote ~6 GB of evicted residual lines
// to DRAM per TD n=8192 side).  Otherwise the residual row is `work`.
// No minimum-blocks hint: ptxas then keeps <= 64 registers (two 512-thread
// CTAs per SM); an explicit hint of 1 lets it take ~88 and costs ~3 ms per TD
// step; 2-4 (forced caps) measured slower too.
template <int K, typename T, int NT, bool SM>
__global__ void __launch_bounds__(NT)
split_rows_kernel(const T* __restrict__ in, size_t in_ld, T* __restrict__ work, size_t cols,
                  int d, int sigma, double* __restrict__ pieces, size_t ldk,
                  size_t slice_stride, unsigned long long* __restrict__ piece_max,
                  int* __restrict__ err, DigitOut dig, bool keep_residual) {
    __shared__ double red[33];
    extern __shared__ double srow_raw[];
    const size_t r = blockIdx.x;
    const T* src = in + r * in_ld * K;
    T* gw = work + r * cols * K;                          // global residual row
    T* w = SM ? reinterpret_cast<T*>(srow_raw) : gw;      // working residual row
    double* prow = pieces ? pieces + r * ldk : nullptr;

    // Sweep 0: leading image max and finiteness scan (ozaki.hpp:77-78).  For
    // D >= 2 the copy of the input row into the working residual is left to
    // pass 0, which reads the input and stores every residual element.
    T mx = T(0);
    int bad = 0;
    if (d == 1 && src != w) {
        for (size_t j = threadIdx.x; j < cols; j += NT) {
            T c[K];
            load_kw<K>(src + j * K, c);
            bad |= !is_finite(c[0]);
            mx = fmax(mx, fabs_(c[0]));
            store_kw<K>(w + j * K, c);
        }
    } else {
        // only the leading words: MultiFloat::is_finite and leading_image look
        // at c[0] alone (multifloat.hpp:176, dense_matrix.hpp:91-96)
        for (size_t j = threadIdx.x; j < cols; j += NT) {
            const T c0 = src[j * K];
            bad |= !is_finite(c0);
            mx = fmax(mx, fabs_(c0));
        }
    }
    if (__syncthreads_or(bad)) {
        if (threadIdx.x == 0) atomicMax(err, (int)kDevNonFinite);
        return;
    }
    mx = (T)block_max((double)mx, red);

    if (d == 1) {
        // D = 1: the piece is the leading image, the residual keeps the tail
        // (ozaki.hpp:90-96: every element, zero or not, gets residual -= lead).
        double pmx = 0.0;
        for (size_t j = threadIdx.x; j < cols; j += NT) {
            T c[K];
            load_kw<K>(w + j * K, c);
            const T lead = c[0];
            if (prow) prow[j] = (double)lead;
            if (keep_residual) {
                kw_add<K>(c, -lead);
                store_kw<K>(gw + j * K, c);
            }
            pmx = fmax(pmx, (double)fabs_(lead));
        }
        if (prow)
            for (size_t j = cols + threadIdx.x; j < ldk; j += NT) prow[j] = 0.0;
        if (piece_max) {
            pmx = block_max(pmx, red);
            if (threadIdx.x == 0)
                atomicMax(piece_max, static_cast<unsigned long long>(__double_as_longlong(pmx)));
        }
        return;
    }

    for (int a = 0; a < d; ++a) {
        double* pa = pieces ? prow + (size_t)a * slice_stride : nullptr;  // optional (INT8 engine)
        T tau = T(0);  // zero marks a skipped (all-zero) row, ozaki.hpp:105-107
        if (mx != T(0)) {
            const int e = ceil_log2(mx);
            if (e + sigma > ShiftGuard<T>::max_exp) {  // ozaki.hpp:109 (mx is block-uniform)
                if (threadIdx.x == 0) atomicMax(err, (int)kDevTooLarge);
                return;
            }
            tau = pow2(T(0), e + sigma);
        }
        T nmx = T(0);
        double pmx = 0.0;
        // the last pass updates the residual only when the caller reads it
        // (ozk_split); the GEMM path drops it (ozaki.hpp:235 never reads it)
        const bool update = keep_residual || a + 1 < d;
        // pass 0 reads the input row; it must store every element when the
        // residual row is a separate buffer (it was not copied in sweep 0)
        const bool store_all = a == 0 && src != w;
        // INT8-digit output: the slice row is an integer multiple of 2^g,
        // g = e + sigma - S: every piece is an integer multiple of this grid
        // (ozaki.hpp:15-29: (v + tau) - tau lands on multiples of ulp of the
        // binade below tau, 2^(e + sigma - S)) with |x| <= 2^e, so
        // |x / 2^g| <= 2^(S - sigma); written as nd signed base-256 digits.
        const int g = (tau == T(0)) ? 0 : (ceil_log2(mx) + sigma - ShiftGuard<T>::S);
        int8_t* drow = dig.digits ? dig.digits + (size_t)a * dig.slice_stride + r * dig.ld : nullptr;
        // 2^-g as a bit-built binary64 when it is normal (x * 2^-g is then the
        // exact integer, no XU-pipe scalbn); scalbn otherwise
        const bool g_normal = -g >= -1022 && -g <= 1023;
        const double inv_grid = g_normal ? __longlong_as_double((long long)(1023 - g) << 52) : 0.0;
        if (dig.digits && threadIdx.x == 0) dig.exps[(size_t)a * dig.exp_stride + r] = g;
        if (tau == T(0)) {  // block-uniform
            for (size_t j = threadIdx.x; j < cols; j += NT) {
                if (pa) pa[j] = 0.0;
                if (drow)
                    for (int q = 0; q < dig.nd; ++q) drow[j + q * dig.digit_stride] = 0;
                if (store_all) {  // skipped row: the residual is the input row
                    T c[K];
                    load_kw<K>(src + j * K, c);
                    store_kw<K>(w + j * K, c);
                }
            }
        } else {
            // rd: the input row (pass 0) or the residual row; compile-time
            // distinct so the shared-memory variant issues LDS/STS
            auto element = [&](size_t j, const T* rd) {
                T c[K];
                load_kw<K>(rd + j * K, c);
                // shift_extract: (v + tau) - tau, strictly rounded (ozaki.hpp:53-56)
                const T x = rn_sub(rn_add(c[0], tau), tau);
                if (pa) pa[j] = (double)x;
                if (drow) {
                    // exact integer; |mi| fits nd digits by the planner's choice of nd
                    int mi = g_normal ? (int)((double)x * inv_grid) : (int)scalbn((double)x, -g);
                    for (int q = 0; q < dig.nd - 1; ++q) {
                        const int dq = (int)(int8_t)(mi & 0xff);
                        drow[j + q * dig.digit_stride] = (int8_t)dq;
                        mi = (mi - dq) >> 8;
                    }
                    drow[j + (dig.nd - 1) * dig.digit_stride] = (int8_t)mi;
                }
                if (update && x != T(0)) {
                    // w -= x  ==  w + (-x)  (multifloat.hpp:304,215), with x the
                    // piece just extracted from w[0] (kword.cuh kw_sub_piece);
                    // FP64 compares: this kernel is ALU-bound, its FP64 pipe
                    // mostly idle
                    kw_sub_piece<K, false>(c, x);
                    store_kw<K>(w + j * K, c);
                } else if (store_all) {
                    store_kw<K>(w + j * K, c);
                }
                nmx = fmax(nmx, fabs_(c[0]));
                pmx = fmax(pmx, (double)fabs_(x));
            };
            // one element per trip: two interleaved per thread measured slower
            // (TD 18.4 -> 22.1 ms, register pressure at 512 threads)
            if (a == 0)
                for (size_t j = threadIdx.x; j < cols; j += NT) element(j, src);
            else
                for (size_t j = threadIdx.x; j < cols; j += NT) element(j, w);
        }
        if (pa)
            for (size_t j = cols + threadIdx.x; j < ldk; j += NT) pa[j] = 0.0;
        if (drow)
            for (size_t j = cols + threadIdx.x; j < dig.ld; j += NT)
                for (int q = 0; q < dig.nd; ++q) drow[j + q * dig.digit_stride] = 0;
        if (piece_max) {
            pmx = block_max(pmx, red);
            if (threadIdx.x == 0)
                atomicMax(piece_max + a,
                          static_cast<unsigned long long>(__double_as_longlong(pmx)));
        }
        if (update) mx = (T)block_max((double)nmx, red);
    }
    if (SM && keep_residual) {  // the caller reads the residual (ozk_split)
        __syncthreads();
        for (size_t j = threadIdx.x; j < cols; j += NT) {
            T c[K];
            load_kw<K>(w + j * K, c);
            store_kw<K>(gw + j * K, c);
        }
    }
}

template <int K, typename T>
__global__ void transpose_kernel(const T* __restrict__ in, size_t in_ld, T* __restrict__ out,
                                 size_t out_ld, size_t rows, size_t cols) {
    __shared__ T tile[32][32 * K + 1];
    const size_t c0 = (size_t)blockIdx.x * 32, r0 = (size_t)blockIdx.y * 32;
    for (int yy = threadIdx.y; yy < 32; yy += 8) {
        const size_t i = r0 + yy;
        if (i >= rows) break;
        const T* src = in + (i * in_ld + c0) * K;
        for (int q = threadIdx.x; q < 32 * K; q += 32)
            if (c0 + q / K < cols) tile[yy][q] = src[q];
    }
    __syncthreads();
    for (int xx = threadIdx.y; xx < 32; xx += 8) {
        const size_t j = c0 + xx;
        if (j >= cols) break;
        T* dst = out + (j * out_ld + r0) * K;
        for (int q = threadIdx.x; q < 32 * K; q += 32) {
            const int yy = q / K, w = q - yy * K;
            if (r0 + yy < rows) dst[q] = tile[yy][xx * K + w];
        }
    }
}

} // namespace

// Shared-memory residual rows: up to this many bytes per row (227 KB per CTA
// minus the reduction scratch), D >= 2; OZK_SPLIT_SMEM=0 forces the global
// variant (A/B builds).
#ifndef OZK_SPLIT_SMEM
#define OZK_SPLIT_SMEM 0
#endif
constexpr size_t kSplitSmemMax = 220 * 1024;
constexpr int kSplitSmemThreads = 1024;

template <int K, typename T>
cudaError_t launch_split_typed(const void* in, size_t in_ld, void* work, size_t rows, size_t cols,
                               int d, int sigma, double* pieces, size_t ldk, size_t slice_stride,
                               unsigned long long* piece_max, int* err, cudaStream_t st,
                               const DigitOut& dig, bool keep_residual) {
    const size_t row_bytes = cols * K * sizeof(T);
    if (OZK_SPLIT_SMEM && d >= 2 && row_bytes <= kSplitSmemMax) {
        auto kern = split_rows_kernel<K, T, kSplitSmemThreads, true>;
        // per call: the attribute belongs to the current device
        const cudaError_t e = cudaFuncSetAttribute(
            kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSplitSmemMax);
        if (e != cudaSuccess) return e;
        kern<<<(unsigned)rows, kSplitSmemThreads, row_bytes, st>>>(
            static_cast<const T*>(in), in_ld, static_cast<T*>(work), cols, d, sigma, pieces, ldk,
            slice_stride, piece_max, err, dig, keep_residual);
    } else {
        split_rows_kernel<K, T, kSplitThreads, false><<<(unsigned)rows, kSplitThreads, 0, st>>>(
            static_cast<const T*>(in), in_ld, static_cast<T*>(work), cols, d, sigma, pieces, ldk,
            slice_stride, piece_max, err, dig, keep_residual);
    }
    return cudaGetLastError();
}

cudaError_t launch_split_rows(int K, int word_bytes, const void* in, size_t in_ld, void* work,
                              size_t rows, size_t cols, int d, int sigma, double* pieces,
                              size_t ldk, size_t slice_stride, unsigned long long* piece_max,
                              int* err, cudaStream_t st, const DigitOut& dig,
                              bool keep_residual) {
    if (rows == 0) return cudaSuccess;
#define OZK_SPLIT(KK, TT)                                                                      \
    launch_split_typed<KK, TT>(in, in_ld, work, rows, cols, d, sigma, pieces, ldk, slice_stride, \
                               piece_max, err, st, dig, keep_residual)
    if (word_bytes == 4) {
        if (K != 3) return cudaErrorInvalidValue;
        return OZK_SPLIT(3, float);
    }
    switch (K) {
    case 2: return OZK_SPLIT(2, double);
    case 3: return OZK_SPLIT(3, double);
    case 4: return OZK_SPLIT(4, double);
    default: return cudaErrorInvalidValue;
    }
#undef OZK_SPLIT
}

cudaError_t launch_transpose(int K, int word_bytes, const void* in, size_t in_ld, void* out,
                             size_t out_ld, size_t rows, size_t cols, cudaStream_t st) {
    if (rows == 0 || cols == 0) return cudaSuccess;
    dim3 grid((unsigned)((cols + 31) / 32), (unsigned)((rows + 31) / 32)), block(32, 8);
#define OZK_TR(KK, TT)                                                                       \
    transpose_kernel<KK, TT><<<grid, block, 0, st>>>(static_cast<const TT*>(in), in_ld,       \
                                                     static_cast<TT*>(out), out_ld, rows, cols)
    if (word_bytes == 4) {
        switch (K) {
        case 1: OZK_TR(1, float); break;
        case 3: OZK_TR(3, float); break;
        default: return cudaErrorInvalidValue;
        }
    } else {
        switch (K) {
        case 1: OZK_TR(1, double); break;
        case 2: OZK_TR(2, double); break;
        case 3: OZK_TR(3, double); break;
        case 4: OZK_TR(4, double); break;
        default: return cudaErrorInvalidValue;
        }
    }
#undef OZK_TR
    return cudaGetLastError();
}

} // namespace ozk
