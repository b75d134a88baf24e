/*
 * ozk_oracle.c -- CPU restatement of the reference Ozaki hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference leg may load this library, and
 * only as the checker (or the timed CPU baseline), never as the product path.
 *
 * This is a plain-C99 restatement of the algorithms in the reference mpmat
 * library (paths relative to /root/reference/proj/include/mpmat/):
 *   eft.hpp:25-39          two_sum, fast_two_sum
 *   multifloat.hpp:34-63 vec_sum, extract_components (VecSumErrBranch)
 *   multifloat.hpp:68-81 canonical_order
 *   multifloat.hpp:159-171 MultiFloat::renormalize
 *   multifloat.hpp:203-213 operator+(MultiFloat, double)
 *   multifloat.hpp:242-257 operator*(MultiFloat, double)
 *   multifloat.hpp:363-430 strict_normalize, from_pair, from_expansion,
 *                          sum_ordered, merge_components
 *   ozaki.hpp:36-56        exponent_ceil_log2, split_shift_bits, shift_extract
 *   ozaki.hpp:74-147       split_matrix
 *   ozaki.hpp:180-249      ozaki_gemm (pair list, drop threshold, accumulation)
 *   rng.hpp:14-54         splitmix64 / xoshiro256** / Box-Muller
 *   gen.hpp:20-34          gen_matrix_eq1
 * It must be compiled with -ffp-contract=off (the reference's own strict-FP
 * flag, proj/CMakeLists.txt:16) and round-to-nearest-even.
 *
 * Parity pinning: tests/test_oracle_golden.py checks this restatement against
 * proj/tests/golden/bench_tiny.csv and eq1_dd_2x2_seed42.mpmat (copied into
 * tests/golden/) and, when oracle/_ref was built from /root/reference,
 * bit-for-bit against the compiled reference itself.
 *
 * Layout conventions (identical to the reference's DenseMatrix<MultiFloat<K>>
 * memory image, dense_matrix.hpp:12-45): a K-word matrix is row-major AoS,
 * element (i,j) word w at ((i*cols + j)*K + w).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define OZK_MAXK 4
#define OZK_MAXTERMS 36 /* max_terms = 2K^2+K for K=4 (multifloat.hpp:133) */

/* ---- eft.hpp:25-39 ------------------------------------------------------ */
static inline void two_sum(double a, double b, double* s, double* e) {
    double ss = a + b;
    double bb = ss - a;
    *e = (a - (ss - bb)) + (b - bb);
    *s = ss;
}

static inline void fast_two_sum(double a, double b, double* s, double* e) {
    double ss = a + b;
    *e = b - (ss - a);
    *s = ss;
}

static inline uint64_t bits_of(double x) {
    uint64_t u;
    memcpy(&u, &x, 8);
    return u;
}

/* ---- multifloat.hpp:34-42 vec_sum -------------------------------------- */
static void vec_sum(double* t, int n) {
    double s = t[n - 1];
    for (int i = n - 2; i >= 0; --i) {
        double hi, lo;
        two_sum(t[i], s, &hi, &lo);
        s = hi;
        t[i + 1] = lo;
    }
    t[0] = s;
}

/* ---- multifloat.hpp:46-63 extract_components<K> ------------------------ */
static void extract_components(int K, const double* t, int n, double* out) {
    for (int i = 0; i < K; ++i) out[i] = 0.0;
    double acc = t[0];
    int j = 0;
    for (int i = 1; i < n; ++i) {
        double hi, lo;
        two_sum(acc, t[i], &hi, &lo);
        if (lo == 0.0) {
            acc = hi;
            continue;
        }
        out[j++] = hi;
        acc = lo;
        if (j == K) return;
    }
    if (j < K) out[j] = acc;
}

/* ---- multifloat.hpp:68-81 canonical_order ------------------------------ */
static void canonical_order(double* t, int n) {
    for (int i = 1; i < n; ++i) {
        double v = t[i];
        double av = fabs(v);
        int j = i - 1;
        while (j >= 0 && (fabs(t[j]) < av || (fabs(t[j]) == av && bits_of(t[j]) > bits_of(v)))) {
            t[j + 1] = t[j];
            --j;
        }
        t[j + 1] = v;
    }
}

/* ---- multifloat.hpp:353-357 non_finite ----------------------------------- */
static void non_finite(int K, double head, double* c) {
    c[0] = head;
    for (int i = 1; i < K; ++i) c[i] = 0.0;
}

/* ---- multifloat.hpp:363-382 strict_normalize ----------------------------- */
static void strict_normalize(int K, double* c) {
    for (int pass = 0; pass < 2 * K; ++pass) {
        int w = 0;
        for (int i = 0; i < K; ++i)
            if (c[i] != 0.0) c[w++] = c[i];
        for (int i = w; i < K; ++i) c[i] = 0.0;
        int changed = 0;
        for (int i = w - 2; i >= 0; --i) {
            double s, e;
            fast_two_sum(c[i], c[i + 1], &s, &e);
            if (s != c[i] || e != c[i + 1]) {
                c[i] = s;
                c[i + 1] = e;
                changed = 1;
            }
        }
        if (!changed) break;
    }
    for (int i = 0; i < K; ++i)
        if (c[i] == 0.0) c[i] = 0.0; /* clear -0 */
}

/* ---- multifloat.hpp:384-392 from_pair (K == 2 only) ---------------------- */
static void from_pair(double s, double e, double* c) {
    if (!isfinite(s)) {
        non_finite(2, s, c);
        return;
    }
    double ps, pe;
    fast_two_sum(s, e, &ps, &pe);
    c[0] = ps == 0.0 ? 0.0 : ps;
    c[1] = (pe == 0.0 || ps == 0.0) ? 0.0 : pe;
}

/* ---- multifloat.hpp:394-401 from_expansion ------------------------------- */
static void from_expansion(int K, const double* t, int n, double* c) {
    extract_components(K, t, n, c);
    strict_normalize(K, c);
    if (c[0] == 0.0 || !isfinite(c[0])) non_finite(K, c[0] + 0.0, c);
}

/* ---- multifloat.hpp:405-416 sum_ordered ---------------------------------- */
static void sum_ordered(int K, const double* t, int n, double* c) {
    double probe = 0.0;
    for (int i = 0; i < n; ++i) probe += t[i];
    if (!isfinite(probe)) {
        non_finite(K, probe, c);
        return;
    }
    double buf[OZK_MAXTERMS > 16 ? OZK_MAXTERMS : 16];
    int m = 0;
    for (int i = 0; i < n; ++i)
        if (t[i] != 0.0) buf[m++] = t[i];
    if (m == 0) {
        for (int i = 0; i < K; ++i) c[i] = 0.0;
        return;
    }
    vec_sum(buf, m);
    from_expansion(K, buf, m, c);
}

/* ---- multifloat.hpp:420-430 merge_components ----------------------------- */
static int before(double x, double y) {
    double ax = fabs(x), ay = fabs(y);
    if (ax != ay) return ax > ay;
    return bits_of(x) <= bits_of(y);
}

static void merge_components(const double* a, int na, const double* b, int nb, double* out) {
    int i = 0, j = 0, k = 0;
    while (i < na && j < nb) out[k++] = before(a[i], b[j]) ? a[i++] : b[j++];
    while (i < na) out[k++] = a[i++];
    while (j < nb) out[k++] = b[j++];
}

/* ---- multifloat.hpp:203-213 operator+(MultiFloat<K>, double) ------------- */
void ozk_oracle_mf_add_double(int K, const double* x, double y, double* r) {
    if (K == 2) {
        double s, e;
        two_sum(x[0], y, &s, &e);
        double v = x[1] + e;
        double fs, fe;
        fast_two_sum(s, v, &fs, &fe);
        from_pair(fs, fe, r);
        return;
    }
    double m[OZK_MAXK + 1];
    merge_components(x, K, &y, 1, m);
    sum_ordered(K, m, K + 1, r);
}

/* ---- multifloat.hpp:159-171 renormalize ---------------------------------- */
static void renormalize(int K, const double* terms, int nterms, double* c) {
    double buf[16] = {0};
    int n = 0;
    double probe = 0.0;
    for (int i = 0; i < nterms; ++i) {
        probe += terms[i];
        if (terms[i] != 0.0) buf[n++] = terms[i];
    }
    if (!isfinite(probe)) {
        non_finite(K, probe, c);
        return;
    }
    if (n == 0) {
        for (int i = 0; i < K; ++i) c[i] = 0.0;
        return;
    }
    vec_sum(buf, n);
    if (n > 1) vec_sum(buf, n);
    from_expansion(K, buf, n, c);
}

/* ---- multifloat.hpp:242-257 operator*(MultiFloat<K>, double) ------------- */
/* two_prod is the FMA form (eft.hpp:60-64, selected at eft.hpp:75-85 when the
 * reference is built with -mfma as its CMakeLists does). */
static void mf_mul_double(int K, const double* x, double y, double* r) {
    if (K == 2) {
        double p = x[0] * y;
        double pe = fma(x[0], y, -p);
        double tail = fma(x[1], y, pe);
        double fs, fe;
        fast_two_sum(p, tail, &fs, &fe);
        from_pair(fs, fe, r);
        return;
    }
    double terms[2 * OZK_MAXK];
    int n = 0;
    for (int i = 0; i < K; ++i) {
        double p = x[i] * y;
        terms[n++] = p;
        terms[n++] = fma(x[i], y, -p);
    }
    canonical_order(terms, n);
    sum_ordered(K, terms, n, r);
}

/* ---- rng.hpp:14-54 ------------------------------------------------------- */
typedef struct {
    uint64_t s[4];
} xoshiro;

static uint64_t splitmix64_next(uint64_t* state) {
    uint64_t z = (*state += 0x9e3779b97f4a7c15ULL);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

static void xo_seed(xoshiro* x, uint64_t seed) {
    uint64_t sm = seed;
    for (int i = 0; i < 4; ++i) x->s[i] = splitmix64_next(&sm);
}

static inline uint64_t rotl64(uint64_t v, int k) { return (v << k) | (v >> (64 - k)); }

static uint64_t xo_next(xoshiro* x) {
    uint64_t* s = x->s;
    uint64_t result = rotl64(s[1] * 5, 7) * 9;
    uint64_t t = s[1] << 17;
    s[2] ^= s[0];
    s[3] ^= s[1];
    s[1] ^= s[2];
    s[0] ^= s[3];
    s[2] ^= t;
    s[3] = rotl64(s[3], 45);
    return result;
}

static double xo_uniform(xoshiro* x) { return (double)(xo_next(x) >> 11) * 0x1p-53; }

static double xo_normal(xoshiro* x) {
    double u1 = xo_uniform(x);
    double u2 = xo_uniform(x);
    double r = sqrt(-2.0 * log(1.0 - u1));
    return r * cos(2.0 * 3.141592653589793 * u2);
}

/* ---- gen.hpp:20-34 gen_matrix_eq1<K> -------------------------------------- */
void ozk_oracle_gen_eq1(int K, size_t m, size_t n, uint64_t seed, double* out) {
    xoshiro rng;
    xo_seed(&rng, seed);
    double comp[OZK_MAXK], ru[OZK_MAXK], t[OZK_MAXK];
    for (size_t idx = 0; idx < m * n; ++idx) {
        for (int k = 0; k < K; ++k) comp[k] = scalbn(xo_uniform(&rng), -53 * k);
        renormalize(K, comp, K, ru);
        double scale = exp(xo_normal(&rng));
        ozk_oracle_mf_add_double(K, ru, -0.5, t); /* ru - 0.5 == ru + (-0.5) (multifloat.hpp:215) */
        mf_mul_double(K, t, scale, out + idx * (size_t)K);
    }
}

/* Raw xoshiro256** stream, for golden checks of the generator itself. */
void ozk_oracle_xoshiro_u64(uint64_t seed, size_t count, uint64_t* out) {
    xoshiro rng;
    xo_seed(&rng, seed);
    for (size_t i = 0; i < count; ++i) out[i] = xo_next(&rng);
}

/* ---- ozaki.hpp:36-56 ------------------------------------------------------ */
int ozk_oracle_exponent_ceil_log2(double x) {
    int e = ilogb(x);
    return scalbn(1.0, e) == x ? e : e + 1;
}

int ozk_oracle_split_shift_bits(size_t inner, int short_bits) {
    int cl = 0;
    while (((size_t)1 << cl) < inner) ++cl;
    return (short_bits + cl + 1) / 2;
}

static double shift_extract(double v, double tau) {
    volatile double shifted = v + tau;
    return shifted - tau;
}

/* ---- ozaki.hpp:74-147 split_matrix<K> ------------------------------------- *
 * side 0 = rows (left factor A, per-row scaling), 1 = cols (right factor B).
 * pieces: d planes of rows*cols doubles, row-major (the reference layout).
 * residual: K-word AoS rows*cols.  Returns 0, or 2 (param_error) for d < 1,
 * a non-finite entry, or "entries too large to shift". */
int ozk_oracle_split(int K, size_t rows, size_t cols, const double* mat, int d, int side,
                     double* pieces, double* residual) {
    if (d < 1) return 2;
    const size_t N = rows * cols;
    for (size_t i = 0; i < N; ++i)
        if (!isfinite(mat[i * K])) return 2; /* MultiFloat::is_finite looks at c[0] */
    const size_t inner = side == 0 ? cols : rows;
    const size_t outer = side == 0 ? rows : cols;
    const int sigma = ozk_oracle_split_shift_bits(inner, 53);
    memcpy(residual, mat, N * (size_t)K * sizeof(double));

    if (d == 1) {
        for (size_t i = 0; i < N; ++i) {
            double lead = residual[i * K];
            pieces[i] = lead;
            double r[OZK_MAXK];
            ozk_oracle_mf_add_double(K, residual + i * K, -lead, r);
            memcpy(residual + i * K, r, (size_t)K * sizeof(double));
        }
        return 0;
    }

    double* mu = (double*)malloc(outer * sizeof(double));
    double* tau = (double*)malloc(outer * sizeof(double));
    int status = 0;
    for (int alpha = 0; alpha < d && status == 0; ++alpha) {
        double* piece = pieces + (size_t)alpha * N;
        /* leading image + per-row/col max (dense_matrix.hpp:72-96) */
        for (size_t o = 0; o < outer; ++o) mu[o] = 0.0;
        for (size_t i = 0; i < rows; ++i)
            for (size_t j = 0; j < cols; ++j) {
                size_t o = side == 0 ? i : j;
                mu[o] = fmax(mu[o], fabs(residual[(i * cols + j) * K]));
            }
        for (size_t o = 0; o < outer; ++o) {
            tau[o] = 0.0;
            if (mu[o] == 0.0) continue;
            int e = ozk_oracle_exponent_ceil_log2(mu[o]);
            if (e + sigma > 1020) {
                status = 2;
                break;
            }
            tau[o] = scalbn(1.0, e + sigma);
        }
        if (status) break;
        for (size_t i = 0; i < rows; ++i)
            for (size_t j = 0; j < cols; ++j) {
                size_t o = side == 0 ? i : j;
                size_t e = i * cols + j;
                if (tau[o] == 0.0) {
                    piece[e] = 0.0;
                    continue;
                }
                double x = shift_extract(residual[e * K], tau[o]);
                piece[e] = x;
                if (x != 0.0) {
                    double r[OZK_MAXK];
                    ozk_oracle_mf_add_double(K, residual + e * K, -x, r);
                    memcpy(residual + e * K, r, (size_t)K * sizeof(double));
                }
            }
    }
    free(mu);
    free(tau);
    return status;
}

/* Binary64 product C = A*B of split pieces, with an exactness witness: every
 * partial product and partial sum is checked to be error-free (TwoProd via
 * fma, TwoSum), so a nonzero return means the split did NOT make the product
 * exact.  The GemmBackend contract (backend.hpp:8-11) allows any order. */
long ozk_oracle_exact_dgemm(size_t m, size_t l, size_t n, const double* A, const double* B,
                            double* C) {
    long inexact = 0;
    for (size_t i = 0; i < m; ++i)
        for (size_t j = 0; j < n; ++j) {
            double s = 0.0;
            int bad = 0;
            for (size_t k = 0; k < l; ++k) {
                double a = A[i * l + k], b = B[k * n + j];
                double p = a * b;
                if (fma(a, b, -p) != 0.0) bad = 1;
                double hi, lo;
                two_sum(s, p, &hi, &lo);
                if (lo != 0.0) bad = 1;
                s = hi;
            }
            C[i * n + j] = s;
            inexact += bad;
        }
    return inexact;
}

/* Plain binary64 GEMM (any-order contract), for the GemmBackend parity check. */
void ozk_oracle_dgemm(size_t m, size_t l, size_t n, const double* A, const double* B, double* C) {
    for (size_t i = 0; i < m; ++i) {
        for (size_t j = 0; j < n; ++j) C[i * n + j] = 0.0;
        for (size_t k = 0; k < l; ++k) {
            double a = A[i * l + k];
            for (size_t j = 0; j < n; ++j) C[i * n + j] += a * B[k * n + j];
        }
    }
}

static double piece_max(const double* p, size_t N) {
    double m = 0.0;
    for (size_t i = 0; i < N; ++i) m = fmax(m, fabs(p[i]));
    return m;
}

/* ---- ozaki.hpp:198-221 pair list ----------------------------------------- *
 * Writes the (alpha, beta) pairs in reference order into pairs[2*P]; returns P. */
int ozk_oracle_pair_list(int d, const double* amax, const double* bmax, double drop,
                         int* pairs) {
    const double lead = amax[0] * bmax[0];
    int np = 0;
    for (int a = 0; a < d; ++a)
        for (int b = 0; a + b < d; ++b) {
            if (drop > 0.0 && amax[a] * bmax[b] < drop * lead) continue;
            pairs[2 * np] = a;
            pairs[2 * np + 1] = b;
            ++np;
        }
    return np;
}

/* ---- ozaki.hpp:180-249 ozaki_gemm<K> -------------------------------------- *
 * Returns 0, 1 (shape_error), 2 (param_error), 5 (out of memory).  Products
 * are formed one pair at a time (exact in any order, so identical to the
 * reference's materialised products) and accumulated in the reference's
 * alpha-major pair order with operator+(MultiFloat, double).  inexact_out,
 * if non-NULL, receives the number of C_ab entries that were NOT error-free. */
int ozk_oracle_ozaki_gemm(int K, size_t m, size_t l, size_t n, const double* A,
                          const double* B, int d, double drop, double* C, int* npairs_out,
                          long* inexact_out) {
    if (d < 1) return 2;
    if (drop < 0.0) return 2;
    const size_t NA = m * l, NB = l * n, NC = m * n;
    double* pa = (double*)malloc((size_t)d * NA * sizeof(double));
    double* pb = (double*)malloc((size_t)d * NB * sizeof(double));
    double* ra = (double*)malloc(NA * (size_t)K * sizeof(double));
    double* rb = (double*)malloc(NB * (size_t)K * sizeof(double));
    double* prod = (double*)malloc(NC * sizeof(double));
    int* pairs = (int*)malloc(sizeof(int) * 2 * (size_t)d * (size_t)d);
    double* amax = (double*)malloc(sizeof(double) * (size_t)d);
    double* bmax = (double*)malloc(sizeof(double) * (size_t)d);
    int st = 0;
    if (!pa || !pb || !ra || !rb || !prod || !pairs || !amax || !bmax) st = 5;
    if (!st) st = ozk_oracle_split(K, m, l, A, d, 0, pa, ra);
    if (!st) st = ozk_oracle_split(K, l, n, B, d, 1, pb, rb);
    if (!st) {
        for (int i = 0; i < d; ++i) {
            amax[i] = piece_max(pa + (size_t)i * NA, NA);
            bmax[i] = piece_max(pb + (size_t)i * NB, NB);
        }
        int np = ozk_oracle_pair_list(d, amax, bmax, drop, pairs);
        if (npairs_out) *npairs_out = np;
        for (size_t e = 0; e < NC * (size_t)K; ++e) C[e] = 0.0;
        long inexact = 0;
        for (int p = 0; p < np; ++p) {
            inexact += ozk_oracle_exact_dgemm(m, l, n, pa + (size_t)pairs[2 * p] * NA,
                                              pb + (size_t)pairs[2 * p + 1] * NB, prod);
            for (size_t e = 0; e < NC; ++e) {
                double r[OZK_MAXK];
                ozk_oracle_mf_add_double(K, C + e * K, prod[e], r);
                memcpy(C + e * K, r, (size_t)K * sizeof(double));
            }
        }
        if (inexact_out) *inexact_out = inexact;
    }
    free(pa);
    free(pb);
    free(ra);
    free(rb);
    free(prod);
    free(pairs);
    free(amax);
    free(bmax);
    return st;
}

/* Sampled-element replay of C for large problems: given the slices (A pieces
 * row-major m x l, B pieces row-major l x n) and the pair list, recomputes
 * C(i,j) for the listed elements exactly as the reference does.  Cost is
 * O(P * l) per element, so n = 8192 checks are cheap. */
void ozk_oracle_replay_elements(int K, size_t m, size_t l, size_t n, const double* pa,
                                const double* pb, int npairs, const int* pairs, size_t count,
                                const long* ii, const long* jj, double* out, long* inexact) {
    long bad = 0;
    for (size_t s = 0; s < count; ++s) {
        double acc[OZK_MAXK] = {0, 0, 0, 0};
        for (int p = 0; p < npairs; ++p) {
            const double* a = pa + (size_t)pairs[2 * p] * m * l + (size_t)ii[s] * l;
            const double* b = pb + (size_t)pairs[2 * p + 1] * l * n + (size_t)jj[s];
            double sum = 0.0;
            for (size_t k = 0; k < l; ++k) {
                double pr = a[k] * b[k * n];
                if (fma(a[k], b[k * n], -pr) != 0.0) ++bad;
                double hi, lo;
                two_sum(sum, pr, &hi, &lo);
                if (lo != 0.0) ++bad;
                sum = hi;
            }
            double r[OZK_MAXK];
            ozk_oracle_mf_add_double(K, acc, sum, r);
            memcpy(acc, r, sizeof(double) * (size_t)K);
        }
        memcpy(out + s * K, acc, sizeof(double) * (size_t)K);
    }
    if (inexact) *inexact = bad;
}

/* ======================================================================== *
 * TS (triple-single): NOT in the reference (MultiFloat<K> is
 * static_assert-ed to binary64 words, multifloat.hpp:129).  The paper uses a
 * 3 x binary32 "triple-single" format.  Following SURVEY
 * §8c, TS is defined here by restating the reference's GENERIC K >= 3
 * algorithms with binary32 words and S = 24:
 *   eft.hpp:25-39 (two_sum, fast_two_sum) in float;
 *   multifloat.hpp:203-213 (K >= 3 branch: merge_components -> sum_ordered),
 *   :121-150 (vec_sum, extract_components), :450-469 (strict_normalize),
 *   :246-260 (renormalize) with K = 3 float words;
 *   ozaki.hpp:36-147 with S = 24 (sigma = (24 + ceil(log2 l) + 1) / 2), a
 *   float volatile shift, and the "too large to shift" guard at e + sigma > 124
 *   (the binary64 guard 1020 keeps 3 binades below the 1023 maximum exponent;
 *   binary32's maximum is 127).
 * Parity for TS is therefore "unpinned by the reference": it is pinned against
 * this restatement (GPU bit-exact) and against the exact big-int oracle
 * (tests/test_ts.py: slices exact, C within the stated ulp bound).
 * ======================================================================== */

static inline uint32_t fbits_of(float x) {
    uint32_t u;
    memcpy(&u, &x, 4);
    return u;
}

static inline void two_sum_f(float a, float b, float* s, float* e) {
    float ss = a + b;
    float bb = ss - a;
    *e = (a - (ss - bb)) + (b - bb);
    *s = ss;
}

static inline void fast_two_sum_f(float a, float b, float* s, float* e) {
    float ss = a + b;
    *e = b - (ss - a);
    *s = ss;
}

static void vec_sum_f(float* t, int n) {
    float s = t[n - 1];
    for (int i = n - 2; i >= 0; --i) {
        float hi, lo;
        two_sum_f(t[i], s, &hi, &lo);
        s = hi;
        t[i + 1] = lo;
    }
    t[0] = s;
}

static void extract_components_f(const float* t, int n, float* out) {
    for (int i = 0; i < 3; ++i) out[i] = 0.0f;
    float acc = t[0];
    int j = 0;
    for (int i = 1; i < n; ++i) {
        float hi, lo;
        two_sum_f(acc, t[i], &hi, &lo);
        if (lo == 0.0f) {
            acc = hi;
            continue;
        }
        out[j++] = hi;
        acc = lo;
        if (j == 3) return;
    }
    if (j < 3) out[j] = acc;
}

static void strict_normalize_f(float* c) {
    for (int pass = 0; pass < 6; ++pass) {
        int w = 0;
        for (int i = 0; i < 3; ++i)
            if (c[i] != 0.0f) c[w++] = c[i];
        for (int i = w; i < 3; ++i) c[i] = 0.0f;
        int changed = 0;
        for (int i = w - 2; i >= 0; --i) {
            float s, e;
            fast_two_sum_f(c[i], c[i + 1], &s, &e);
            if (s != c[i] || e != c[i + 1]) {
                c[i] = s;
                c[i + 1] = e;
                changed = 1;
            }
        }
        if (!changed) break;
    }
    for (int i = 0; i < 3; ++i)
        if (c[i] == 0.0f) c[i] = 0.0f;
}

static void from_expansion_f(const float* t, int n, float* c) {
    extract_components_f(t, n, c);
    strict_normalize_f(c);
    if (c[0] == 0.0f || !isfinite(c[0])) {
        c[0] = c[0] + 0.0f;
        c[1] = c[2] = 0.0f;
    }
}

static void sum_ordered_f(const float* t, int n, float* c) {
    float probe = 0.0f;
    for (int i = 0; i < n; ++i) probe += t[i];
    if (!isfinite(probe)) {
        c[0] = probe;
        c[1] = c[2] = 0.0f;
        return;
    }
    float buf[16];
    int m = 0;
    for (int i = 0; i < n; ++i)
        if (t[i] != 0.0f) buf[m++] = t[i];
    if (m == 0) {
        c[0] = c[1] = c[2] = 0.0f;
        return;
    }
    vec_sum_f(buf, m);
    from_expansion_f(buf, m, c);
}

static int before_f(float x, float y) {
    float ax = fabsf(x), ay = fabsf(y);
    if (ax != ay) return ax > ay;
    return fbits_of(x) <= fbits_of(y);
}

/* TS + float: the K >= 3 branch of multifloat.hpp:203-213 with float words. */
void ozk_oracle_ts_add_float(const float* x, float y, float* r) {
    float m[4];
    int i = 0, k = 0, placed = 0;
    while (i < 3 && !placed) {
        if (before_f(x[i], y))
            m[k++] = x[i++];
        else {
            m[k++] = y;
            placed = 1;
        }
    }
    while (i < 3) m[k++] = x[i++];
    if (!placed) m[k++] = y;
    sum_ordered_f(m, 4, r);
}

static void renormalize_f(const float* terms, int nterms, float* c) {
    float buf[16] = {0};
    int n = 0;
    float probe = 0.0f;
    for (int i = 0; i < nterms; ++i) {
        probe += terms[i];
        if (terms[i] != 0.0f) buf[n++] = terms[i];
    }
    if (!isfinite(probe)) {
        c[0] = probe;
        c[1] = c[2] = 0.0f;
        return;
    }
    if (n == 0) {
        c[0] = c[1] = c[2] = 0.0f;
        return;
    }
    vec_sum_f(buf, n);
    if (n > 1) vec_sum_f(buf, n);
    from_expansion_f(buf, n, c);
}

/* TS inputs: Eq. (1) TD values (gen_matrix_eq1<3>, gen.hpp:20-34) rounded to
 * three binary32 words by successive leading-word extraction in binary64,
 * then renormalised in TS (renormalize, multifloat.hpp:159-171). */
void ozk_oracle_gen_eq1_ts(size_t m, size_t n, uint64_t seed, float* out) {
    double* td = (double*)malloc(m * n * 3 * sizeof(double));
    ozk_oracle_gen_eq1(3, m, n, seed, td);
    for (size_t e = 0; e < m * n; ++e) {
        const double* c = td + 3 * e;
        float w[3];
        double r0 = c[0];
        w[0] = (float)r0;
        double r1 = (r0 - (double)w[0]) + c[1];
        w[1] = (float)r1;
        double r2 = ((r1 - (double)w[1]) + c[2]);
        w[2] = (float)r2;
        renormalize_f(w, 3, out + 3 * e);
    }
    free(td);
}

int ozk_oracle_exponent_ceil_log2_f(float x) {
    int e = ilogbf(x);
    return scalbnf(1.0f, e) == x ? e : e + 1;
}

static float shift_extract_f(float v, float tau) {
    volatile float shifted = v + tau;
    return shifted - tau;
}

/* TS split: ozaki.hpp:74-147 with S = 24 (see block comment above). */
int ozk_oracle_split_ts(size_t rows, size_t cols, const float* mat, int d, int side,
                        float* pieces, float* residual) {
    if (d < 1) return 2;
    const size_t N = rows * cols;
    for (size_t i = 0; i < N; ++i)
        if (!isfinite(mat[i * 3])) return 2;
    const size_t inner = side == 0 ? cols : rows;
    const size_t outer = side == 0 ? rows : cols;
    const int sigma = ozk_oracle_split_shift_bits(inner, 24);
    memcpy(residual, mat, N * 3 * sizeof(float));
    if (d == 1) {
        for (size_t i = 0; i < N; ++i) {
            float lead = residual[i * 3];
            pieces[i] = lead;
            float r[3];
            ozk_oracle_ts_add_float(residual + i * 3, -lead, r);
            memcpy(residual + i * 3, r, sizeof r);
        }
        return 0;
    }
    float* mu = (float*)malloc(outer * sizeof(float));
    float* tau = (float*)malloc(outer * sizeof(float));
    int status = 0;
    for (int alpha = 0; alpha < d && status == 0; ++alpha) {
        float* piece = pieces + (size_t)alpha * N;
        for (size_t o = 0; o < outer; ++o) mu[o] = 0.0f;
        for (size_t i = 0; i < rows; ++i)
            for (size_t j = 0; j < cols; ++j) {
                size_t o = side == 0 ? i : j;
                mu[o] = fmaxf(mu[o], fabsf(residual[(i * cols + j) * 3]));
            }
        for (size_t o = 0; o < outer; ++o) {
            tau[o] = 0.0f;
            if (mu[o] == 0.0f) continue;
            int e = ozk_oracle_exponent_ceil_log2_f(mu[o]);
            if (e + sigma > 124) {
                status = 2;
                break;
            }
            tau[o] = scalbnf(1.0f, e + sigma);
        }
        if (status) break;
        for (size_t i = 0; i < rows; ++i)
            for (size_t j = 0; j < cols; ++j) {
                size_t o = side == 0 ? i : j;
                size_t e = i * cols + j;
                if (tau[o] == 0.0f) {
                    piece[e] = 0.0f;
                    continue;
                }
                float x = shift_extract_f(residual[e * 3], tau[o]);
                piece[e] = x;
                if (x != 0.0f) {
                    float r[3];
                    ozk_oracle_ts_add_float(residual + e * 3, -x, r);
                    memcpy(residual + e * 3, r, sizeof r);
                }
            }
    }
    free(mu);
    free(tau);
    return status;
}

/* binary32 slice product with an exactness witness (TwoProd via fmaf, TwoSum). */
long ozk_oracle_exact_sgemm(size_t m, size_t l, size_t n, const float* A, const float* B,
                            float* C) {
    long inexact = 0;
    for (size_t i = 0; i < m; ++i)
        for (size_t j = 0; j < n; ++j) {
            float s = 0.0f;
            int bad = 0;
            for (size_t k = 0; k < l; ++k) {
                float a = A[i * l + k], b = B[k * n + j];
                float p = a * b;
                if (fmaf(a, b, -p) != 0.0f) bad = 1;
                float hi, lo;
                two_sum_f(s, p, &hi, &lo);
                if (lo != 0.0f) bad = 1;
                s = hi;
            }
            C[i * n + j] = s;
            inexact += bad;
        }
    return inexact;
}

/* TS Ozaki GEMM: ozaki.hpp:180-249 over the TS split and binary32 products. */
int ozk_oracle_ozaki_gemm_ts(size_t m, size_t l, size_t n, const float* A, const float* B, int d,
                             double drop, float* C, int* npairs_out, long* inexact_out) {
    if (d < 1 || drop < 0.0) return 2;
    const size_t NA = m * l, NB = l * n, NC = m * n;
    float* pa = (float*)malloc((size_t)d * NA * sizeof(float));
    float* pb = (float*)malloc((size_t)d * NB * sizeof(float));
    float* ra = (float*)malloc(NA * 3 * sizeof(float));
    float* rb = (float*)malloc(NB * 3 * sizeof(float));
    float* prod = (float*)malloc(NC * sizeof(float));
    int* pairs = (int*)malloc(sizeof(int) * 2 * (size_t)d * (size_t)d);
    double* amax = (double*)malloc(sizeof(double) * (size_t)d);
    double* bmax = (double*)malloc(sizeof(double) * (size_t)d);
    int st = 0;
    if (!pa || !pb || !ra || !rb || !prod || !pairs || !amax || !bmax) st = 5;
    if (!st) st = ozk_oracle_split_ts(m, l, A, d, 0, pa, ra);
    if (!st) st = ozk_oracle_split_ts(l, n, B, d, 1, pb, rb);
    if (!st) {
        for (int i = 0; i < d; ++i) {
            float ma = 0.0f, mb = 0.0f;
            for (size_t e = 0; e < NA; ++e) ma = fmaxf(ma, fabsf(pa[(size_t)i * NA + e]));
            for (size_t e = 0; e < NB; ++e) mb = fmaxf(mb, fabsf(pb[(size_t)i * NB + e]));
            amax[i] = ma;
            bmax[i] = mb;
        }
        int np = ozk_oracle_pair_list(d, amax, bmax, drop, pairs);
        if (npairs_out) *npairs_out = np;
        for (size_t e = 0; e < NC * 3; ++e) C[e] = 0.0f;
        long inexact = 0;
        for (int p = 0; p < np; ++p) {
            inexact += ozk_oracle_exact_sgemm(m, l, n, pa + (size_t)pairs[2 * p] * NA,
                                              pb + (size_t)pairs[2 * p + 1] * NB, prod);
            for (size_t e = 0; e < NC; ++e) {
                float r[3];
                ozk_oracle_ts_add_float(C + e * 3, prod[e], r);
                memcpy(C + e * 3, r, sizeof r);
            }
        }
        if (inexact_out) *inexact_out = inexact;
    }
    free(pa);
    free(pb);
    free(ra);
    free(rb);
    free(prod);
    free(pairs);
    free(amax);
    free(bmax);
    return st;
}

/* ---- direct TS GEMM (the config-4 comparator; no reference counterpart) ----
 * C(i,j) = sum_k A(i,k) * B(k,j) in triple-single arithmetic, k ascending,
 * one multiply-accumulate per term (the paper's GPU "direct" TS GEMM,
 * PAPER.md:280-312, TwoProd/TwoSum in binary32).  This is its definition; the
 * GPU kernel (csrc/ts_direct.cu) replays it bit for bit.
 *   product, truncated below level 2 (|term| ~ u^2 |a0 b0|):
 *     (p00,e00) = TwoProd(a0,b0); (p01,e01) = TwoProd(a0,b1); (p10,e10) = TwoProd(a1,b0)
 *     t2 = ((a0*b2 + a1*b1) + a2*b0) + (e01 + e10)
 *   accumulate into (s0,s1,s2):
 *     (s0,r0) = TwoSum(s0,p00); (q,r1) = TwoSum(p01,p10); (q,r2) = TwoSum(q,e00)
 *     (s1,r3) = TwoSum(s1,q);   (s1,r4) = TwoSum(s1,r0)
 *     s2 = (((s2 + t2) + r1) + r2) + (r3 + r4)
 *   renormalise: (s1,s2) = TwoSum(s1,s2); (s0,s1) = TwoSum(s0,s1); (s1,s2) = TwoSum(s1,s2)
 */
void ozk_oracle_ts_fma(float* s, const float* a, const float* b) {
    float p00 = a[0] * b[0], e00 = fmaf(a[0], b[0], -p00);
    float p01 = a[0] * b[1], e01 = fmaf(a[0], b[1], -p01);
    float p10 = a[1] * b[0], e10 = fmaf(a[1], b[0], -p10);
    float t2 = ((a[0] * b[2] + a[1] * b[1]) + a[2] * b[0]) + (e01 + e10);
    float s0, r0, q, r1, r2, s1, r3, r4;
    two_sum_f(s[0], p00, &s0, &r0);
    two_sum_f(p01, p10, &q, &r1);
    two_sum_f(q, e00, &q, &r2);
    two_sum_f(s[1], q, &s1, &r3);
    two_sum_f(s1, r0, &s1, &r4);
    float s2 = (((s[2] + t2) + r1) + r2) + (r3 + r4);
    two_sum_f(s1, s2, &s1, &s2);
    two_sum_f(s0, s1, &s0, &s1);
    two_sum_f(s1, s2, &s1, &s2);
    s[0] = s0;
    s[1] = s1;
    s[2] = s2;
}

void ozk_oracle_ts_direct_gemm(size_t m, size_t l, size_t n, const float* A, const float* B,
                               float* C) {
    for (size_t i = 0; i < m; ++i)
        for (size_t j = 0; j < n; ++j) {
            float s[3] = {0.0f, 0.0f, 0.0f};
            for (size_t k = 0; k < l; ++k)
                ozk_oracle_ts_fma(s, A + (i * l + k) * 3, B + (k * n + j) * 3);
            C[(i * n + j) * 3 + 0] = s[0];
            C[(i * n + j) * 3 + 1] = s[1];
            C[(i * n + j) * 3 + 2] = s[2];
        }
}

/* ---- ill-conditioned inputs (BASELINE config 5) -----------------------------
 * Eq. (1) elements (gen.hpp:20-34, same per-element draws) each scaled by 2^e,
 * e uniform on [-spread, spread] drawn from the same stream right after the
 * element's Eq. (1) draws -- the exponent-spread idea of random_scaled
 * (proj/tests/acceptance.cpp:53-58) applied to K-word values.  Scaling by a
 * power of two is exact, so every element keeps its full K*53-bit significand
 * while rows span up to 2*spread binades. */
void ozk_oracle_gen_spread(int K, size_t m, size_t n, uint64_t seed, int spread, double* out) {
    xoshiro rng;
    xo_seed(&rng, seed);
    double comp[OZK_MAXK], ru[OZK_MAXK], t[OZK_MAXK];
    for (size_t idx = 0; idx < m * n; ++idx) {
        for (int k = 0; k < K; ++k) comp[k] = scalbn(xo_uniform(&rng), -53 * k);
        renormalize(K, comp, K, ru);
        double scale = exp(xo_normal(&rng));
        ozk_oracle_mf_add_double(K, ru, -0.5, t);
        double* o = out + idx * (size_t)K;
        mf_mul_double(K, t, scale, o);
        int e = (int)(xo_next(&rng) % (uint64_t)(2 * spread + 1)) - spread;
        for (int k = 0; k < K; ++k) o[k] = scalbn(o[k], e);
    }
}
