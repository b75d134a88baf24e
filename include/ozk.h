/*
 * ozk.h -- C-ABI of the B200 Ozaki-scheme multiple-precision GEMM.
 *
 * This is the drop-in boundary for the reference mpmat library's hot path
 * (paths relative to /root/reference/proj/include/mpmat/):
 *
 *   ozk_ozaki_gemm        replaces  template<int K> ozaki_gemm(a, b, d, backend,
 *                                   drop_threshold)                  ozaki.hpp:180-183
 *   ozk_split             replaces  template<int K> split_matrix(m, d, side)
 *                                                                    ozaki.hpp:74-75
 *   ozk_backend_gemm      replaces  reference_backend_gemm / the GemmBackend plugin
 *                                                                    backend.hpp:12-20
 *   ozk_split_shift_bits  replaces  split_shift_bits                 ozaki.hpp:43-48
 *   ozk_exponent_ceil_log2 replaces exponent_ceil_log2               ozaki.hpp:36-40
 *
 * Conventions (identical to the reference, so the boundary is zero-copy):
 *  - matrices are row-major; a K-word element is K consecutive doubles
 *    (the memory image of DenseMatrix<MultiFloat<K>>, dense_matrix.hpp:12-45,
 *    multifloat.hpp:131): element (i,j) word w at ((i*cols + j)*K + w);
 *  - the split count is `int split_count` (>= 1), the component type is the
 *    ozk_format (K = 2/3/4 words = DD/TD/QD);
 *  - no exception crosses the ABI: every call returns an ozk_status and
 *    ozk_last_error() (thread-local) describes the last failure.  The status
 *    codes map 1:1 onto the reference's exception types (errors.hpp:7-25) and
 *    are raised for the same conditions in the same order.  A null matrix
 *    pointer (which the reference's references cannot express) is refused
 *    with OZK_EPARAM after those checks, before any device work.
 *
 * All functions are reentrant (the reference calls its backend from an
 * OpenMP parallel loop, ozaki.hpp:224-231); host-buffer entry points use a
 * private CUDA stream per call.  `*_device` entry points take device
 * pointers and a cudaStream_t (passed as void*, NULL = legacy default
 * stream) and synchronise that stream before returning.
 */
#ifndef OZK_H
#define OZK_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    OZK_OK = 0,
    OZK_ESHAPE = 1, /* mpmat::shape_error  (errors.hpp:11-13) */
    OZK_EPARAM = 2, /* mpmat::param_error  (errors.hpp:15-17) */
    OZK_ECUDA = 3,  /* CUDA runtime / launch failure */
    OZK_ENCCL = 4,  /* collective failure (multi-GPU entry points) */
    OZK_ENOMEM = 5, /* device allocation failure */
    OZK_EIO = 6     /* mpmat::io_error     (errors.hpp:23-25), MPMAT file I/O */
} ozk_status;

/* Element format.  DD/TD/QD: K = 2/3/4 binary64 words, = the reference's
 * MultiFloat<K> template argument.  TS (triple-single): 3 binary32 words per
 * element -- not in the reference; defined by restating its
 * generic K >= 3 algorithms with binary32 words and S = 24 (oracle/ozk_oracle.c).
 * Matrix buffers are void*: K words of the format's word type per element. */
typedef enum { OZK_DD = 2, OZK_TD = 3, OZK_QD = 4, OZK_TS = 0x103 } ozk_format;

/* mpmat::SplitSide (ozaki.hpp:33) */
typedef enum { OZK_SIDE_ROWS = 0, OZK_SIDE_COLS = 1 } ozk_side;

/* superset of mpmat::OzakiProfile (ozaki.hpp:149-167).  product_seconds covers
 * the fused slice-GEMM + accumulation kernel; accumulate_seconds is 0 when the
 * accumulation is fused (always, today).  total = split + product + accumulate
 * as in the reference; transfer_seconds (host entry points only) is the
 * host<->device copy time, outside total. */
typedef struct {
    double split_seconds;
    double product_seconds;
    double accumulate_seconds;
    double total_seconds;
    double transfer_seconds;
    int split_count;
    int pairs;
    int gpus;
    int engine; /* ozk_engine that formed the slice products */
} ozk_profile;

/* Slice-product engine.  Both give bit-identical C (every slice product is
 * exact either way):
 *   DMMA : FP64 tensor cores (mma.sync m8n8k4.f64), any shape;
 *   INT8 : each FP64 slice is an integer on its row/column power-of-two grid
 *          (|M| <= 2^(53-sigma)); for 128 < l < 43690 it is split into 3 signed
 *          int8 digits and the 9 digit GEMMs run on tcgen05.mma kind::i8 with
 *          exact int32 accumulation in TMEM (csrc/gemm_i8.cu);
 *   AUTO : INT8 where it applies (DD/TD/QD, D >= 2, 128 < l < 43690; TS
 *          l < 43690), else DMMA. */
typedef enum { OZK_ENGINE_AUTO = 0, OZK_ENGINE_DMMA = 1, OZK_ENGINE_INT8 = 2 } ozk_engine;
ozk_status ozk_set_engine(int engine); /* process-wide; default from $OZK_ENGINE */
int ozk_get_engine(void);

/* ---- the reference entry points ------------------------------------------ */

/* C (m x n) = A (m x l) * B (l x n) in K-word precision via the Ozaki scheme
 * (ozaki.hpp:180-249): host buffers.  Errors, in the reference's order:
 * OZK_ESHAPE for a zero dimension (dense_matrix.hpp:23) or mismatched inner
 * dimensions (ozaki.hpp:184), OZK_EPARAM for split_count < 1 (:185),
 * drop_threshold < 0 (:186), a non-finite entry (:77-78) or an entry too
 * large to shift (:109).  Any split_count >= 1 (slice indices are 16-bit:
 * up to 65535; device memory, D slice planes per side, is the practical
 * limit); pair lists longer than one launch run as consecutive launches. */
ozk_status ozk_ozaki_gemm(ozk_format fmt, size_t m, size_t l, size_t n, const void* a,
                          const void* b, int split_count, double drop_threshold, void* c,
                          ozk_profile* prof);

/* Same with device-resident a, b, c on `stream`. */
ozk_status ozk_ozaki_gemm_device(ozk_format fmt, size_t m, size_t l, size_t n, const void* a,
                                 const void* b, int split_count, double drop_threshold, void* c,
                                 void* stream, ozk_profile* prof);

/* Asynchronous ozk_ozaki_gemm_device for pipelined callers: returns once the
 * work is queued on `stream` (scratch is stream-ordered).  The split's data
 * errors (non-finite entry, entry too large to shift; A's, then B's) land in
 * dev_flags[0..1], two device ints read with ozk_check_split_flag (A's flag
 * first, as the reference splits A first); the return value covers argument
 * and launch errors.  With drop_threshold > 0 the pair list needs the slice
 * maxima on the host, so that case synchronises once mid-call and returns a
 * data error directly, as ozk_ozaki_gemm_device does. */
ozk_status ozk_ozaki_gemm_device_async(ozk_format fmt, size_t m, size_t l, size_t n,
                                       const void* a, const void* b, int split_count,
                                       double drop_threshold, void* c, int* dev_flags,
                                       void* stream);

/* split_matrix<K> (ozaki.hpp:74-147): host buffers.  pieces receives
 * split_count row-major (rows x cols) slices (binary64; binary32 for TS),
 * residual the K-word working matrix after the last extraction (SplitSet<K>,
 * ozaki.hpp:59-67). */
ozk_status ozk_split(ozk_format fmt, size_t rows, size_t cols, const void* mat, int split_count,
                     ozk_side side, void* pieces, void* residual);

/* GemmBackend (backend.hpp:12-13): C = A * B in binary64, row-major, host
 * buffers.  Any summation order (the plugin contract, backend.hpp:8-11). */
ozk_status ozk_backend_gemm(size_t m, size_t l, size_t n, const double* a, const double* b,
                            double* c);
ozk_status ozk_backend_gemm_device(size_t m, size_t l, size_t n, const double* a,
                                   const double* b, double* c, void* stream);

int ozk_split_shift_bits(size_t inner_dim);  /* ozaki.hpp:43-48 */
int ozk_exponent_ceil_log2(double x);        /* ozaki.hpp:36-40 (x > 0, finite) */

/* ---- slice-level entry points (sharded / multi-GPU orchestration) --------- *
 * Slices are kept in the DMMA operand layout: split_count planes of `outer`
 * rows of ozk_slice_ld(inner) doubles (k contiguous, zero padded; TS slices
 * are binary32 values stored exactly as binary64).
 *   side ROWS (left factor A, m x l):  slices[a][i][k] = piece_a(i, k)
 *   side COLS (right factor B, l x n): slices[a][j][k] = piece_a(k, j)
 * `ld` is the row stride (in elements) of the input K-word matrix, so a
 * column block of B can be split in place.  Slice planes are plane_rows
 * (>= outer) rows apart, so a ragged last column block keeps the padded
 * block layout; rows past `outer` are left untouched.  piece_max (nullable) receives
 * max|piece_a| per slice (for drop_threshold, ozaki.hpp:198-208), combined by
 * max with whatever it held (zero-fill it first). */
size_t ozk_slice_ld(size_t inner_dim);

ozk_status ozk_split_slices_device(ozk_format fmt, size_t rows, size_t cols, size_t ld,
                                   const void* mat, int split_count, ozk_side side,
                                   double* slices, size_t plane_rows, double* piece_max,
                                   void* stream);

/* Pair list of ozaki.hpp:198-221 (alpha-major, triangular, drop pruning).
 * pairs receives 2*npairs ints (alpha, beta); capacity split_count^2 ints. */
ozk_status ozk_pair_list(int split_count, const double* amax, const double* bmax,
                         double drop_threshold, int* pairs, int* npairs);

/* Fused slice-pair GEMMs + K-word accumulation (ozaki.hpp:223-244) over
 * precomputed slices.  a_slices: split_count x m x ozk_slice_ld(l).  The B
 * slices may be stored in nblk column blocks of ncb columns each (the layout an
 * all-gather of column-sharded B slices produces): column j = blk*ncb + jj is
 * at b_slices + blk*b_blk_stride + beta*ncb*ld + jj*ld (ld = ozk_slice_ld(l)).
 * Pass nblk = 1, ncb = n for a single block.  c is m x n K-word, row stride
 * ldc elements; it is overwritten. */
ozk_status ozk_slices_gemm_device(ozk_format fmt, size_t m, size_t l, size_t n,
                                  const double* a_slices, const double* b_slices, size_t ncb,
                                  size_t nblk, size_t b_blk_stride, int split_count,
                                  const int* pairs, int npairs, void* c, size_t ldc,
                                  void* stream);

/* ---- automatic split count (not in the reference) ------------- *
 * A policy for (split_count, drop_threshold) from the format and the inner
 * dimension alone: enough slices to capture the full K-word significand,
 * D = ceil(S*K / (S - sigma)) + 2 (S = 53, or 24 for TS), and the
 * reference's own pair pruning (ozaki.hpp:198-221) at
 * drop = 2^-(S*K + ceil(log2 l) + 2): pairs whose products are normwise below
 * the format's precision are skipped.  ozk_ozaki_gemm(..., D, drop, ...) with
 * these values equals the reference's ozaki_gemm(a, b, D, backend, drop) bit
 * for bit; for Eq. (1) inputs at l = 8192 it keeps the pairs of the measured
 * accuracy saturation (DD 7, TD 9, QD 12). */
int ozk_auto_split_count(ozk_format fmt, size_t inner_dim);
double ozk_auto_drop_threshold(ozk_format fmt, size_t inner_dim);

/* ---- INT8-digit slice entry points (sharded orchestration, INT8 engine) ---- *
 * The exact INT8 engine stores each slice as nd signed base-256 digit planes of
 * the slice integers plus one grid exponent per row (A) / column (B):
 *   piece_a(i, k) = 2^exps[a][i] * sum_t 256^t * digits[a][t][i][k]
 * digits: split_count x nd x plane_rows x ld8 int8 (ld8 >= inner dimension, a
 * multiple of 16, zero padded), exps: split_count x plane_rows ints.  nd is
 * ozk_int8_digits(fmt, inner, split_count); 0 means the engine does not apply
 * (binary64 slices at inner dimension <= 128, or inner >= 43690).  The products
 * and the K-word accumulation are bit-identical to ozk_slices_gemm_device. */
int ozk_int8_digits(ozk_format fmt, size_t inner_dim, int split_count);

ozk_status ozk_split_digits_device(ozk_format fmt, size_t rows, size_t cols, size_t ld,
                                   const void* mat, int split_count, ozk_side side,
                                   int8_t* digits, size_t ld8, size_t plane_rows, int* exps,
                                   double* piece_max, void* stream);

/* Asynchronous forms for pipelined callers (sharded.py): nothing is
 * synchronised.  The split reports data errors (non-finite entry, too large to
 * shift) through *dev_flag, a device int the caller zero-fills first and
 * checks with ozk_check_split_flag (which synchronises `stream`); the return
 * value covers argument and launch errors only.  Scratch is stream-ordered. */
ozk_status ozk_split_digits_device_async(ozk_format fmt, size_t rows, size_t cols, size_t ld,
                                         const void* mat, int split_count, ozk_side side,
                                         int8_t* digits, size_t ld8, size_t plane_rows, int* exps,
                                         double* piece_max, int* dev_flag, void* stream);
ozk_status ozk_check_split_flag(const int* dev_flag, void* stream);
ozk_status ozk_digits_gemm_device_async(ozk_format fmt, size_t m, size_t l, size_t n,
                                        const int8_t* a_digits, const int* a_exps,
                                        size_t a_plane_rows, const int8_t* b_digits,
                                        const int* b_exps, size_t b_plane_rows, size_t ld8,
                                        int split_count, const int* pairs, int npairs, void* c,
                                        size_t ldc, void* stream);

/* Fused INT8 slice-pair GEMMs + K-word accumulation over digit planes: A digits
 * for m rows (a_plane_rows >= m), B digits for n columns (b_plane_rows >= n),
 * both with row length ld8; c is m x n K-word, row stride ldc, overwritten. */
ozk_status ozk_digits_gemm_device(ozk_format fmt, size_t m, size_t l, size_t n,
                                  const int8_t* a_digits, const int* a_exps, size_t a_plane_rows,
                                  const int8_t* b_digits, const int* b_exps, size_t b_plane_rows,
                                  size_t ld8, int split_count, const int* pairs, int npairs,
                                  void* c, size_t ldc, void* stream);

/* ---- MPMAT v1 matrix files (proj/src/matrix_io.cpp) ---------- *
 * Text: header "MPMAT v1 <tag> <m> <n>", then one matrix row per line, each
 * element as its K words in C99 hex ("%a", space separated).  Tags d, dd, td,
 * qd (fmt OZK_D = 1, OZK_DD, OZK_TD, OZK_QD) as in the reference, plus "ts"
 * (OZK_TS, 3 binary32 words; this build's extension, each word written as the
 * equal binary64 literal and read back exactly).  Round trips are bit-exact and
 * the written bytes equal the reference writer's.  a: m x n elements of K words
 * (float words for TS), row-major.  Errors: OZK_EIO with the reference's
 * io_error messages (unopenable file, bad header, not MPMAT v1, tag mismatch,
 * zero dimension, truncated row, malformed element). */
#define OZK_D 1
ozk_status ozk_mpmat_write(const char* path, int fmt, size_t m, size_t n, const void* a);
ozk_status ozk_mpmat_read_header(const char* path, int* fmt, size_t* m, size_t* n);
ozk_status ozk_mpmat_read(const char* path, int fmt, size_t m, size_t n, void* a);

/* The reference's accumulation phase on its own (ozaki.hpp:235-244): for each
 * element, acc = 0; acc += products[p] for p = 0..nproducts-1 in order, with
 * MultiFloat<K> + double; c receives the m x n K-word result (binary32 words
 * for TS, each product rounded to binary32 first -- exact for TS slice
 * products).  For callers that form the slice products with their own
 * GemmBackend (mpmat::gpu::ozaki_gemm with a foreign backend).  Host version:
 * products[p] are m x n row-major host arrays; device version: one contiguous
 * nproducts x m x n device array. */
ozk_status ozk_accumulate_products(ozk_format fmt, size_t m, size_t n,
                                   const double* const* products, int nproducts, void* c);
ozk_status ozk_accumulate_products_device(ozk_format fmt, size_t m, size_t n,
                                          const double* products, int nproducts, void* c,
                                          void* stream);

/* Parity hook: every slice product C_ab = A_alpha * B_beta of the pair list,
 * binary64, into products[p] (m x n row-major). */
ozk_status ozk_pair_products_device(size_t m, size_t l, size_t n, const double* a_slices,
                                    const double* b_slices, int split_count, const int* pairs,
                                    int npairs, double* products, void* stream);

/* Parity hook of the INT8 engine: every slice product C_ab of the pair list,
 * formed exactly as the INT8 slice GEMM forms it (nd^2 int8 digit GEMMs on
 * tcgen05 with int32 accumulation, exact int64 recombination, scaling by
 * 2^(gA + gB)), stored as binary64 into products[p] (m x n row-major) instead
 * of being accumulated.  Operands as for ozk_digits_gemm_device. */
ozk_status ozk_pair_products_digits_device(ozk_format fmt, size_t m, size_t l, size_t n,
                                           const int8_t* a_digits, const int* a_exps,
                                           size_t a_plane_rows, const int8_t* b_digits,
                                           const int* b_exps, size_t b_plane_rows, size_t ld8,
                                           int split_count, const int* pairs, int npairs,
                                           double* products, void* stream);

/* ---- blocked-LU trailing update ------------------- *
 * A22 := A22 - L21 * U12 exactly as the reference's blocked_lu does it
 * (proj/include/mpmat/lu.hpp:104-124): the product by ozaki_gemm with
 * split_count slices, then A22(i,j) -= update(i,j) with MultiFloat<K>
 * subtraction (multifloat.hpp:300,201).  L21: tm x pw (row stride ldl), U12:
 * pw x tn (row stride ldu), A22: tm x tn (row stride lda), all in elements,
 * so the blocks can live inside the full matrix.  DD/TD/QD only. */
ozk_status ozk_lu_trailing_update(ozk_format fmt, size_t tm, size_t pw, size_t tn,
                                  const void* l21, size_t ldl, const void* u12, size_t ldu,
                                  void* a22, size_t lda, int split_count);
ozk_status ozk_lu_trailing_update_device(ozk_format fmt, size_t tm, size_t pw, size_t tn,
                                         const void* l21, size_t ldl, const void* u12,
                                         size_t ldu, void* a22, size_t lda, int split_count,
                                         void* stream);

/* ---- multi-GPU, one process (SURVEY §8b ozk_ozaki_gemm_multi, §8e) -------- *
 * ozk_ozaki_gemm on ngpus devices (devices[r], or 0..ngpus-1 when devices is
 * NULL) from host buffers, one host thread per device: device r owns C rows
 * [r*m/ngpus, (r+1)*m/ngpus), splits its A rows and its B column block (per-row
 * / per-column splits = the global split, ozaki.hpp:102-103), the B digit
 * planes are all-gathered by peer copies (NVLink), slice maxima are combined
 * on the host when drop > 0, and each device runs all pairs for its rows and
 * copies its C rows back.  C is bit-identical to ozk_ozaki_gemm for any
 * ngpus.  Where the INT8 engine does not apply (or DMMA is forced) each device
 * runs ozk_ozaki_gemm on its rows against the whole B.  A device may repeat in
 * `devices` (the kernels of different entries never wait on each other).
 * prof (optional): total_seconds = slowest device, pairs, gpus, engine. */
ozk_status ozk_ozaki_gemm_multi(ozk_format fmt, int ngpus, const int* devices, size_t m, size_t l,
                                size_t n, const void* a, const void* b, int split_count,
                                double drop_threshold, void* c, ozk_profile* prof);

/* ---- host-buffer schedule (introspection) --------------------------------- *
 * The row bands ozk_ozaki_gemm's overlapped host path uses for an m x n C on
 * the INT8 engine, planned from the slice GEMM's tile geometry: group_rows /
 * group_cols C rows / columns per cluster tile, `clusters` co-resident clusters
 * of cluster_sms SMs each, B arriving in column blocks of block_cols.  Writes
 * up to max_bands + 1 row starts (0, ..., m) to starts and returns the number
 * of bands, or -1 (bad arguments / more than max_bands bands).  Pure host
 * function; no GPU needed.  No reference counterpart (this build's schedule). */
int ozk_plan_row_bands(ozk_format fmt, size_t m, size_t n, size_t l, int split_count,
                       size_t block_cols, int group_rows, int group_cols, int clusters,
                       int cluster_sms, size_t* starts, int max_bands);

/* ---- direct K-word GEMM -------------------------------------- *
 * The reference's gemm_simple<MultiFloat<K>> (gemm.hpp:15-31) bit for bit:
 * per element c = 0; for k ascending: c = c + a(i,k) * b(k,j) with the
 * reference's K-word multiply (multifloat.hpp:218-239) and add (:184-199).
 * The comparator the Ozaki scheme is measured against (paper §5); DD/TD/QD,
 * row-major AoS, a: m x l, b: l x n, c: m x n. */
ozk_status ozk_direct_gemm(ozk_format fmt, size_t m, size_t l, size_t n, const void* a,
                           const void* b, void* c);
ozk_status ozk_direct_gemm_device(ozk_format fmt, size_t m, size_t l, size_t n, const void* a,
                                  const void* b, void* c, void* stream);

/* ---- direct triple-single GEMM (BASELINE config 4 comparator) ------------- *
 * C = A * B with every term accumulated in triple-single arithmetic, k
 * ascending (no reference counterpart; the operation sequence is defined in
 * oracle/ozk_oracle.c: ozk_oracle_ts_fma).  a: m x l, b: l x n, c: m x n,
 * 3 binary32 words per element, row-major. */
ozk_status ozk_ts_direct_gemm(size_t m, size_t l, size_t n, const float* a, const float* b,
                              float* c);
ozk_status ozk_ts_direct_gemm_device(size_t m, size_t l, size_t n, const float* a,
                                     const float* b, float* c, void* stream);

/* ---- utilities -------------------------------------------------------------- */

/* The reference's input generator gen_matrix_eq1<K>(rows, cols, seed)
 * (gen.hpp:20-34, Xoshiro256ss rng.hpp:21-54) into a HOST buffer, bit for bit:
 * the same single xoshiro256** stream, entered by every worker thread at its
 * first element by a GF(2) jump (csrc/gen_host.cpp), and the same libm calls.
 * threads <= 0: all CPUs this process may run on.  TS: the TD value rounded
 * to three binary32 words and renormalised (this build's TS definition). */
ozk_status ozk_gen_eq1(ozk_format fmt, size_t rows, size_t cols, uint64_t seed, void* out,
                       int threads);

/* Ill-conditioned inputs (BASELINE config 5, acceptance.cpp:53-58 style): each
 * gen_matrix_eq1 element scaled by 2^e, e uniform on [-spread, spread] from one
 * further draw of the same stream (0 <= spread <= 400). */
ozk_status ozk_gen_spread(ozk_format fmt, size_t rows, size_t cols, uint64_t seed, int spread,
                          void* out, int threads);

/* Eq. (1)-distributed synthetic K-word matrix (rows*cols elements) in device
 * memory; counter-based, so a pure function of (seed, shape).  Not the
 * reference's sequential generator (gen.hpp:20-34) -- see csrc/gen.cu. */
ozk_status ozk_gen_eq1_device(ozk_format fmt, size_t rows, size_t cols, uint64_t seed,
                              void* out, void* stream);

/* Ill-conditioned variant (BASELINE config 5): the same elements scaled by
 * 2^e, e uniform on [-spread, spread] (0 <= spread <= 400). */
ozk_status ozk_gen_spread_device(ozk_format fmt, size_t rows, size_t cols, uint64_t seed,
                                 int spread, void* out, void* stream);

/* FP64 tensor-pipe (DMMA) ceiling of the current device in TFLOP/s, measured by a
 * register-resident mma.sync.m8n8k4.f64 loop on every SM (the roofline
 * denominator for the slice GEMMs).  Returns < 0 on failure. */
double ozk_probe_dmma_tflops(int iters, void* stream);

/* Dense INT8 tensor ceiling (tcgen05.mma kind::i8, M=128 N=256, one CTA per SM,
 * operands resident in shared memory) in TOPS -- the INT8 engine's roofline
 * denominator.  Returns < 0 on failure. */
double ozk_probe_i8_tops(int iters, void* stream);

/* Scratch comes from the current device's stream-ordered pool, which keeps
 * freed memory for the next call (release threshold: never).  This returns
 * the pool's unused memory to the device, for callers that need it for other
 * allocators.  Synchronises the device. */
ozk_status ozk_trim_device_pool(void);

const char* ozk_last_error(void);
int ozk_version(void);

#ifdef __cplusplus
}
#endif

#endif /* OZK_H */
