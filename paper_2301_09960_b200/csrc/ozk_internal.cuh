// ozk_internal.cuh -- launchers shared between the kernel TUs and the C-ABI TU.
#pragma once

#include <string>
#include <vector>

#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

namespace ozk {

// Split counts: slice indices are 16-bit in the kernels' pair lists; the
// reference itself only requires d >= 1 (ozaki.hpp:185).  Memory (D slices per
// side) is the practical limit long before this.
constexpr int kMaxSplits = 65535;
// Pairs per kernel launch (the pair list travels in the kernel parameter
// block); longer lists run as consecutive launches that continue the K-word
// accumulation in C, so the per-element pair order is unchanged.
constexpr int kPairsPerLaunch = 528;

// Device-side error flags raised by the split kernel (read back by the host),
// combined with atomicMax: a non-finite entry anywhere outranks an entry too
// large to shift, as the reference scans the whole matrix for finiteness before
// any shift (ozaki.hpp:77-78 before :109).
enum DevErr : int { kDevOk = 0, kDevTooLarge = 1, kDevNonFinite = 2 };

// Leading dimension (doubles) of a slice row: the inner dimension rounded up to
// 16 bytes, as TMA requires 16-byte global strides.  Pad entries are zero.
inline size_t slice_ld(size_t inner) { return (inner + 1) & ~size_t(1); }

// K1: per-row Ozaki split of a K-word matrix (ozaki.hpp:74-147, side rows).
//   in      : rows x cols K-word AoS, row stride in_ld elements (may alias work)
//   work    : rows x cols K-word AoS scratch (row stride cols); holds the residual
//             after the last pass only when keep_residual (else its last pass
//             update is skipped: the GEMM path never reads it)
//   pieces  : d slices, slice a row r at pieces + a*slice_stride + r*ldk
//   piece_max (optional): d values, max |piece_a| as ordered uint64 bits
//   err     : device flag (DevErr)
// Optional INT8-digit output of the split (for the exact INT8 slice-product
// engine): slice a, row r has grid exponent exps[a*exp_stride + r] = g and
// digits[a*slice_stride + s*digit_stride + r*ld + k], s = 0..nd-1, with
// piece(r, k) = 2^g * sum_s 256^s d_s, g = e + sigma - (S + 1) (S = 53 for
// binary64 words, 24 for TS).  digits == nullptr: off.
struct DigitOut {
    int nd = 3;     // digits written per element (1..3)
    int8_t* digits = nullptr;
    size_t ld = 0, digit_stride = 0, slice_stride = 0;
    int* exps = nullptr;
    size_t exp_stride = 0;
};

// word_bytes = 8 for DD/TD/QD (binary64 words), 4 for TS (binary32 words, K = 3).
cudaError_t launch_split_rows(int K, int word_bytes, const void* in, size_t in_ld, void* work,
                              size_t rows, size_t cols, int d, int sigma, double* pieces,
                              size_t ldk, size_t slice_stride, unsigned long long* piece_max,
                              int* err, cudaStream_t st, const DigitOut& dig = DigitOut{},
                              bool keep_residual = true);

// Transpose of a K-word matrix: out(j, i) = in(i, j).  in is rows x cols with
// row stride in_ld elements; out is cols x rows with row stride out_ld elements.
cudaError_t launch_transpose(int K, int word_bytes, const void* in, size_t in_ld, void* out,
                             size_t out_ld, size_t rows, size_t cols, cudaStream_t st);

// Slice-pair GEMM with fused epilogue (K2 + K3).
// kAccumulateLU: kAccumulate whose final pair subtracts the finished sum from
// an A22 block instead of storing it (the blocked-LU trailing update,
// lu.hpp:121-124, fused into the slice-GEMM epilogue)
enum GemmMode : int { kStorePlain = 0, kAccumulate = 1, kStoreProducts = 2, kAccumulateLU = 3 };

// Host-side pair list (alpha-major, ozaki.hpp:210-221), any length.
struct PairList {
    int count = 0;
    std::vector<unsigned short> alpha, beta;
    void clear() {
        count = 0;
        alpha.clear();
        beta.clear();
    }
    void push(int a, int b) {
        alpha.push_back((unsigned short)a);
        beta.push_back((unsigned short)b);
        ++count;
    }
};

// One launch's slice of a PairList (kernel parameter).
struct PairChunk {
    int count;
    unsigned short alpha[kPairsPerLaunch];
    unsigned short beta[kPairsPerLaunch];
};
inline PairChunk pair_chunk(const PairList& pl, int first) {
    PairChunk c;
    c.count = pl.count - first < kPairsPerLaunch ? pl.count - first : kPairsPerLaunch;
    for (int p = 0; p < c.count; ++p) {
        c.alpha[p] = pl.alpha[first + p];
        c.beta[p] = pl.beta[first + p];
    }
    return c;
}

struct GemmProblem {
    // A slices: [d][m][lda] doubles (k contiguous); B^T slices in column blocks:
    // column j lives in block j / ncb at b + blk*b_blk_stride + beta*b_slice_stride
    // + (j % ncb)*ldb.
    const double* a;
    size_t lda, a_slice_stride;
    int a_slices;
    const double* b;
    size_t ldb, b_slice_stride, b_blk_stride;
    int b_slices;
    int ncb, nblk;
    size_t m, n, l;
    void* c;            // K-word AoS of word_bytes words (kAccumulate) or doubles
    size_t ldc;         // elements per row of C
    size_t c_pair_stride;  // kStoreProducts: doubles between consecutive pair products
    uint32_t zero;         // always 0 (runtime value: carries a register dependency)
    uint32_t c_continue;   // kAccumulate: 1 = C already holds a running sum (later pair chunk)
    double* lu_a22;        // kAccumulateLU: A22 block (K-word, row stride lu_lda elements)
    size_t lu_lda;
    uint32_t lu_final;     // kAccumulateLU: this launch holds the list's last pair
};

cudaError_t launch_pair_gemm(int K, GemmMode mode, const GemmProblem& prob, const PairList& pairs,
                             cudaStream_t st, int num_sms, int word_bytes = 8);

// Exact INT8-digit slice products on tcgen05 (gemm_i8.cu).  Digits as written
// by the split's DigitOut: [d][3][rows][ld] int8, exponents [d][rows].
struct I8Operands {
    int nd;         // digits per slice integer (1..3)
    const int8_t* a;
    size_t a_ld, a_digit_stride, a_slice_stride;
    const int8_t* b;
    size_t b_ld, b_digit_stride, b_slice_stride;
    const int* gA;  // [d][gA_stride]
    const int* gB;  // [d][gB_stride]
    size_t gA_stride = 0, gB_stride = 0;  // 0: m / n
    size_t m, n, l;
    int d;
    void* c;        // K-word AoS, row stride ldc elements
    size_t ldc;
    bool c_init = true;      // the first pair starts C from zero (false: accumulate onto C)
    size_t pair_stride = 0;  // launch_pair_products_i8: doubles between pair planes
    // blocked-LU trailing update (binary64 formats): after the list's last pair
    // the sum is subtracted from A22 (row stride lu_lda elements) instead of
    // being stored to C, which then only carries the running sum
    double* lu_a22 = nullptr;
    size_t lu_lda = 0;
};
// Tile geometry of the INT8 slice GEMM for a format: C rows and columns per
// cluster tile and the number of co-resident persistent clusters (one wave =
// `clusters` cluster tiles).  Zeros if the engine does not apply.
struct I8Geometry {
    int group_rows = 0, group_cols = 0, clusters = 0, cluster_sms = 1;
};
I8Geometry pair_gemm_i8_geometry(int K, int word_bytes, int nd, int num_sms);
cudaError_t launch_pair_gemm_i8(int K, int word_bytes, const I8Operands& op,
                                const PairList& pairs, cudaStream_t st, int num_sms);
// Parity hook: every exact slice product C_ab (binary64) into c + p*pair_stride
// (row stride ldc) instead of the K-word accumulation.
cudaError_t launch_pair_products_i8(int word_bytes, const I8Operands& op, const PairList& pairs,
                                    cudaStream_t st, int num_sms);

// Device Eq. (1)-distributed K-word generator (synthetic bench inputs).
// a(i, j) -= c(i, j) in K-word arithmetic (a: row stride lda elements, c dense).
cudaError_t launch_kw_sub_inplace(int K, double* a, size_t lda, const double* c, size_t rows,
                                  size_t cols, cudaStream_t st);

// Accumulation phase on its own (accumulate.cu, ozaki.hpp:235-244): c (count
// K-word elements) = sum over p of prods[p * count + e], in p order.
cudaError_t launch_accumulate_products(int K, int word_bytes, const double* prods, int np,
                                       size_t count, void* c, cudaStream_t st);

// Direct triple-single GEMM (csrc/ts_direct.cu): a (m x l), b (l x n), c (m x n),
// 3 binary32 words per element.
cudaError_t launch_ts_direct(const float* a, const float* b, float* c, size_t m, size_t l,
                             size_t n, cudaStream_t st);

// word_bytes = 4 selects TS (K = 3 binary32 words).
// spread > 0 scales every element by 2^U[-spread, spread] (config 5 inputs).
cudaError_t launch_gen_eq1(int K, int word_bytes, void* out, size_t count, uint64_t seed,
                           int spread, cudaStream_t st);

// Direct K-word GEMM, gemm_simple<MultiFloat<K>> (csrc/direct.cu).
cudaError_t launch_direct_gemm(int K, const double* a, const double* b, double* c, size_t m,
                               size_t l, size_t n, cudaStream_t st);

void set_last_error(const std::string& msg);  // api.cu (ozk_last_error)

// ---- pageable host buffers (staging.cu) -------------------------------------
bool host_is_pinned(const void* p);  // page-locked / registered host memory

// One staged copy: `height` rows of `width` bytes, row pitches dev_pitch /
// host_pitch.  H2D: `event` (optional) is recorded on the H2D stream after the
// copy; D2H: the copy waits for `event` (already recorded) first.
struct StagedCopy {
    void* dev = nullptr;
    void* host = nullptr;
    size_t width = 0, height = 1, dev_pitch = 0, host_pitch = 0;
    cudaEvent_t event = nullptr;
};

// Worker threads moving pageable buffers through pinned slot rings, in
// submission order per direction.  push_h2d returns the job number;
// wait_recorded(job) blocks until that job's event has been recorded (a
// cudaStreamWaitEvent on an unrecorded event would not wait).  finish() drains
// both queues (every D2H job is then in the caller's buffer).
class HostStaging {
public:
    HostStaging(cudaStream_t h2d, cudaStream_t d2h, int h2d_threads, int d2h_threads);
    ~HostStaging();
    int push_h2d(const StagedCopy& c);
    void push_d2h(const StagedCopy& c);
    cudaError_t wait_recorded(int job);
    cudaError_t finish();

private:
    struct Impl;
    Impl* impl_;
    int pushed_h2d_ = 0;
};

} // namespace ozk
