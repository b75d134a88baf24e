// kword.cuh -- K-word (DD/TD/QD) "+ double" for the split and accumulate
// kernels, replaying the reference operation sequence bit for bit.
//
// Reference semantics (paths under /root/reference/proj/include/mpmat/):
//   eft.hpp:25-39            two_sum (Knuth), fast_two_sum (Dekker, no precondition)
//   multifloat.hpp:290-300   operator+(MultiFloat<K>, double)
//                            K=2: two_sum, one add, fast_two_sum, from_pair (:471-479)
//                            K>=3: merge_components (:507-517) -> sum_ordered (:492-503)
//                                  -> vec_sum (:121-129) -> from_expansion (:481-488)
//                                  -> extract_components (:133-150) -> strict_normalize (:450-469)
//
// GPU formulation.  Every array is register resident: all loops are fully
// unrolled with compile-time trip counts and data-dependent positions become
// predicated selects, so nothing spills to local memory.  Two places differ in
// FORM from the reference but not in result:
//   * sum_ordered's zero compaction before vec_sum is skipped.  A zero term
//     is transparent to both sweeps: two_sum(0, s) = (s, 0) leaves the
//     running sum untouched and emits a zero, and extract_components skips
//     zero terms (two_sum(acc, 0) has lo == 0).  The nonzero sequence that
//     reaches extraction is therefore identical, in the same order.
//   * strict_normalize runs its 2K passes unconditionally after the first
//     unchanged pass; a pass with no change is idempotent (compaction finds no
//     interior zero, the sweep finds only fixpoints).
// Both claims are checked bit-for-bit against the compiled reference
// (tests/test_kword_host.py on CPU, tests/test_gpu_parity.py on the GPU).
//
// Only additions/subtractions appear here, so FMA contraction cannot occur;
// the device build still uses the explicit round-to-nearest intrinsics.
#pragma once

#include <stdint.h>

#if defined(__CUDACC__)
#define OZK_HD __host__ __device__ __forceinline__
#else
#define OZK_HD inline
#endif

#if defined(__CUDA_ARCH__)
#define OZK_DADD(a, b) __dadd_rn((a), (b))
#define OZK_DSUB(a, b) __dsub_rn((a), (b))
#else
#define OZK_DADD(a, b) ((a) + (b))
#define OZK_DSUB(a, b) ((a) - (b))
#endif

namespace ozk {

OZK_HD uint64_t dbits(double x) {
#if defined(__CUDA_ARCH__)
    return static_cast<uint64_t>(__double_as_longlong(x));
#else
    union {
        double d;
        uint64_t u;
    } v;
    v.d = x;
    return v.u;
#endif
}

OZK_HD double dabs(double x) {
#if defined(__CUDA_ARCH__)
    return fabs(x);
#else
    return x < 0 ? -x : (x == 0 ? 0.0 : x);
#endif
}

OZK_HD bool dfinite(double x) {
    // exponent field not all ones
    return (dbits(x) & 0x7ff0000000000000ull) != 0x7ff0000000000000ull;
}

// eft.hpp:25-30
OZK_HD void two_sum(double a, double b, double& s, double& e) {
    double ss = OZK_DADD(a, b);
    double bb = OZK_DSUB(ss, a);
    e = OZK_DADD(OZK_DSUB(a, OZK_DSUB(ss, bb)), OZK_DSUB(b, bb));
    s = ss;
}

// eft.hpp:35-39
OZK_HD void fast_two_sum(double a, double b, double& s, double& e) {
    double ss = OZK_DADD(a, b);
    e = OZK_DSUB(b, OZK_DSUB(ss, a));
    s = ss;
}

// multifloat.hpp:509-512 (merge order predicate)
OZK_HD bool merge_before(double x, double y) {
    double ax = dabs(x), ay = dabs(y);
    if (ax != ay) return ax > ay;
    return dbits(x) <= dbits(y);
}

template <int K>
OZK_HD void non_finite(double head, double* c) {
    c[0] = head;
#pragma unroll
    for (int i = 1; i < K; ++i) c[i] = 0.0;
}

// multifloat.hpp:450-469
template <int K>
OZK_HD void strict_normalize(double* c) {
#pragma unroll
    for (int pass = 0; pass < 2 * K; ++pass) {
        // stable compaction of zeros to the tail (bubble, static indices)
#pragma unroll
        for (int r = 0; r < K - 1; ++r) {
#pragma unroll
            for (int i = 0; i < K - 1; ++i) {
                bool z = c[i] == 0.0;
                double lo = c[i + 1];
                c[i + 1] = z ? 0.0 : c[i + 1];
                c[i] = z ? lo : c[i];
            }
        }
        // trailing zeros written by the reference's compaction are +0.0
#pragma unroll
        for (int i = 0; i < K; ++i) c[i] = (c[i] == 0.0) ? 0.0 : c[i];
        bool changed = false;
#pragma unroll
        for (int i = K - 2; i >= 0; --i) {
            double s, e;
            fast_two_sum(c[i], c[i + 1], s, e);
            bool ch = (s != c[i]) || (e != c[i + 1]);
            c[i] = ch ? s : c[i];
            c[i + 1] = ch ? e : c[i + 1];
            changed = changed || ch;
        }
        if (!changed) break;
    }
#pragma unroll
    for (int i = 0; i < K; ++i) c[i] = (c[i] == 0.0) ? 0.0 : c[i];
}

// multifloat.hpp:133-150 over N terms (zero terms are transparent)
template <int K, int N>
OZK_HD void extract_components(const double* t, double* out) {
#pragma unroll
    for (int q = 0; q < K; ++q) out[q] = 0.0;
    double acc = t[0];
    int j = 0;
#pragma unroll
    for (int i = 1; i < N; ++i) {
        if (j < K) {
            double hi, lo;
            two_sum(acc, t[i], hi, lo);
            if (lo == 0.0) {
                acc = hi;
            } else {
#pragma unroll
                for (int q = 0; q < K; ++q) out[q] = (j == q) ? hi : out[q];
                ++j;
                acc = lo;
            }
        }
    }
#pragma unroll
    for (int q = 0; q < K; ++q) out[q] = (j == q) ? acc : out[q];
}

// MultiFloat<K> + double (multifloat.hpp:290-300); x is updated in place.
template <int K>
OZK_HD void kw_add(double* x, double y) {
    if constexpr (K == 2) {
        double s, e;
        two_sum(x[0], y, s, e);
        double v = OZK_DADD(x[1], e);
        double fs, fe;
        fast_two_sum(s, v, fs, fe);
        // from_pair (multifloat.hpp:471-479)
        if (!dfinite(fs)) {
            x[0] = fs;
            x[1] = 0.0;
            return;
        }
        double ps, pe;
        fast_two_sum(fs, fe, ps, pe);
        x[0] = ps == 0.0 ? 0.0 : ps;
        x[1] = (pe == 0.0 || ps == 0.0) ? 0.0 : pe;
    } else {
        // merge_components(x, K, &y, 1): y goes before the first x[i] that
        // does not precede it
        double m[K + 1];
        bool placed = false;
#pragma unroll
        for (int i = 0; i <= K; ++i) {
            bool take_x = !placed && i < K && merge_before(x[i < K ? i : 0], y);
            double prev = x[i > 0 ? i - 1 : 0];
            double cur = x[i < K ? i : K - 1];
            m[i] = placed ? prev : (take_x ? cur : y);
            placed = placed || !take_x;
        }
        // sum_ordered: finiteness probe over all terms
        double probe = 0.0;
#pragma unroll
        for (int i = 0; i <= K; ++i) probe = OZK_DADD(probe, m[i]);
        if (!dfinite(probe)) {
            non_finite<K>(probe, x);
            return;
        }
        // vec_sum over all K+1 terms (zeros transparent, see header)
        double s = m[K];
#pragma unroll
        for (int i = K - 1; i >= 0; --i) {
            double hi, lo;
            two_sum(m[i], s, hi, lo);
            s = hi;
            m[i + 1] = lo;
        }
        m[0] = s;
        // from_expansion
        extract_components<K, K + 1>(m, x);
        strict_normalize<K>(x);
        if (x[0] == 0.0 || !dfinite(x[0])) non_finite<K>(OZK_DADD(x[0], 0.0), x);
    }
}

} // namespace ozk
