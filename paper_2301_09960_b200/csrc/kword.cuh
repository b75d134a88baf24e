// kword.cuh -- K-word (DD/TD/QD) "+ double" for the split and accumulate
// kernels, replaying the reference operation sequence bit for bit.
//
// Reference semantics (paths under /root/reference/proj/include/mpmat/):
//   eft.hpp:25-39            two_sum (Knuth), fast_two_sum (Dekker, no precondition)
//   multifloat.hpp:203-213   operator+(MultiFloat<K>, double)
//                            K=2: two_sum, one add, fast_two_sum, from_pair (:384-392)
//                            K>=3: merge_components (:420-430) -> sum_ordered (:405-416)
//                                  -> vec_sum (:34-42) -> from_expansion (:394-401)
//                                  -> extract_components (:46-63) -> strict_normalize (:363-382)
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
//     interior zero, the sweep finds only fixpoints).  On the K >= 3 fast path the
//     first pass also skips its zero compaction: from_expansion's output has
//     no interior zero (see kw_add_impl).
// These claims are checked bit-for-bit against the compiled reference
// (tests/test_kword_host.py on CPU, tests/test_gpu_parity.py on the GPU).
//
// Only additions/subtractions appear here, so FMA contraction cannot occur;
// the device build still uses the explicit round-to-nearest intrinsics.
#pragma once

#include <stdint.h>
#if !defined(__CUDACC__)
#include <cmath>
#endif

#if defined(__CUDACC__)
#define OZK_HD __host__ __device__ __forceinline__
#else
#define OZK_HD inline
#endif

namespace ozk {

// ---- scalar primitives, overloaded for binary64 (DD/TD/QD) and binary32 (TS) ----

OZK_HD double rn_add(double a, double b) {
#if defined(__CUDA_ARCH__)
    return __dadd_rn(a, b);
#else
    return a + b;
#endif
}
OZK_HD double rn_sub(double a, double b) {
#if defined(__CUDA_ARCH__)
    return __dsub_rn(a, b);
#else
    return a - b;
#endif
}
OZK_HD float rn_add(float a, float b) {
#if defined(__CUDA_ARCH__)
    return __fadd_rn(a, b);
#else
    return a + b;
#endif
}
OZK_HD float rn_sub(float a, float b) {
#if defined(__CUDA_ARCH__)
    return __fsub_rn(a, b);
#else
    return a - b;
#endif
}

OZK_HD uint64_t fbits(double x) {
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
OZK_HD uint32_t fbits(float x) {
#if defined(__CUDA_ARCH__)
    return static_cast<uint32_t>(__float_as_uint(x));
#else
    union {
        float f;
        uint32_t u;
    } v;
    v.f = x;
    return v.u;
#endif
}
// kept for the split/gemm call sites
OZK_HD uint64_t dbits(double x) { return fbits(x); }

OZK_HD double fabs_(double x) {
#if defined(__CUDA_ARCH__)
    return fabs(x);
#else
    return x < 0 ? -x : (x == 0 ? 0.0 : x);
#endif
}
OZK_HD float fabs_(float x) {
#if defined(__CUDA_ARCH__)
    return fabsf(x);
#else
    return x < 0 ? -x : (x == 0 ? 0.0f : x);
#endif
}
OZK_HD double dabs(double x) { return fabs_(x); }

// exponent field not all ones
OZK_HD bool is_finite(double x) {
    return (fbits(x) & 0x7ff0000000000000ull) != 0x7ff0000000000000ull;
}
OZK_HD bool is_finite(float x) { return (fbits(x) & 0x7f800000u) != 0x7f800000u; }
OZK_HD bool dfinite(double x) { return is_finite(x); }

// ---- comparisons -------------------------------------------------------------
// kInt = false: the reference's floating-point comparisons.  kInt = true: the
// same predicates on the bit patterns (integer ALU instead of DSETP on the FP64
// pipe, which the tensor cores share on sm_100).  They agree for every finite
// operand whose words stay below 2^1000 (2^120 for binary32), which kw_add's
// guard (kw_fast_ok) checks before taking that path: no NaN (where FP and bit
// comparisons differ), no overflow to infinity inside the sweeps, and -0 never
// reaches a bitwise comparison (the compaction writes +0; x - x rounds to +0).
template <typename T> struct Bits;
template <> struct Bits<double> {
    using U = uint64_t;
    static constexpr U kAbs = 0x7fffffffffffffffull;
    static constexpr U kSafe = (uint64_t)(1023 + 1000) << 52;  // |x| < 2^1000
};
template <> struct Bits<float> {
    using U = uint32_t;
    static constexpr U kAbs = 0x7fffffffu;
    static constexpr U kSafe = (uint32_t)(127 + 120) << 23;     // |x| < 2^120
};

// 32-bit halves: the high word carries sign + exponent (+ top significand)
OZK_HD uint32_t hi_word(double x) { return (uint32_t)(fbits(x) >> 32); }
OZK_HD uint32_t lo_word(double x) { return (uint32_t)fbits(x); }
OZK_HD uint32_t hi_word(float x) { return fbits(x); }
OZK_HD uint32_t lo_word(float) { return 0u; }

// The kInt predicates work on the 32-bit halves: a 64-bit sign mask is
// recognised by the compiler as |x| and issued as an FP64 DADD, which is
// exactly the pipe (shared with the tensor cores on sm_100) these avoid.
template <bool kInt, typename T>
OZK_HD bool is_zero(T x) {
    if constexpr (kInt) return ((hi_word(x) & 0x7fffffffu) | lo_word(x)) == 0u;
    else return x == T(0);
}
template <bool kInt, typename T>
OZK_HD bool same(T a, T b) {  // a == b in the kInt domain described above
    if constexpr (kInt) return hi_word(a) == hi_word(b) && lo_word(a) == lo_word(b);
    else return a == b;
}

// eft.hpp:25-30
template <typename T>
OZK_HD void two_sum(T a, T b, T& s, T& e) {
    T ss = rn_add(a, b);
    T bb = rn_sub(ss, a);
    e = rn_add(rn_sub(a, rn_sub(ss, bb)), rn_sub(b, bb));
    s = ss;
}

// eft.hpp:35-39
template <typename T>
OZK_HD void fast_two_sum(T a, T b, T& s, T& e) {
    T ss = rn_add(a, b);
    e = rn_sub(b, rn_sub(ss, a));
    s = ss;
}

// multifloat.hpp:421-425 (merge order predicate)
template <bool kInt = false, typename T>
OZK_HD bool merge_before(T x, T y) {
    if constexpr (kInt) {
        // |x| vs |y| on the magnitude bits (monotone for non-NaN values),
        // lexicographic over (high word without sign, low word)
        const uint32_t hx = hi_word(x) & 0x7fffffffu, hy = hi_word(y) & 0x7fffffffu;
        const uint32_t lx = lo_word(x), ly = lo_word(y);
        if (hx != hy || lx != ly) return hx > hy || (hx == hy && lx > ly);
        // equal magnitudes: raw-bit order puts +x before -x
        return hi_word(x) <= hi_word(y);
    } else {
        T ax = fabs_(x), ay = fabs_(y);
        if (ax != ay) return ax > ay;
    }
    return fbits(x) <= fbits(y);
}

template <int K, typename T>
OZK_HD void non_finite(T head, T* c) {
    c[0] = head;
#pragma unroll
    for (int i = 1; i < K; ++i) c[i] = T(0);
}

// multifloat.hpp:363-382
// OZK_KW_TAILSKIP=0 keeps the first compaction on the fast path (A/B builds).
#ifndef OZK_KW_TAILSKIP
#define OZK_KW_TAILSKIP 1
#endif

// OZK_KW_ZGUARD=0 runs the compaction unconditionally (A/B builds).
#ifndef OZK_KW_ZGUARD
#define OZK_KW_ZGUARD 1
#endif

// kTailZeros: the caller guarantees c has no zero before a nonzero word, so
// the first pass's compaction is the identity and is skipped.
template <int K, bool kInt = false, bool kTailZeros = false, typename T>
OZK_HD void strict_normalize(T* c) {
#pragma unroll
    for (int pass = 0; pass < 2 * K; ++pass) {
        // stable compaction of zeros to the tail (bubble, static indices).  It
        // is the identity unless a zero sits before the last word (a zero in
        // the last word is already at the tail), so it runs only then: the
        // common case costs K-1 zero tests instead of 2(K-1)^2 selects.
        bool interior_zero = !OZK_KW_ZGUARD;
#pragma unroll
        for (int i = 0; i < K - 1; ++i) interior_zero = interior_zero || is_zero<kInt>(c[i]);
        if (interior_zero) {
#pragma unroll
            for (int r = 0; r < ((kTailZeros && pass == 0) ? 0 : K - 1); ++r) {
#pragma unroll
                for (int i = 0; i < K - 1; ++i) {
                    bool z = is_zero<kInt>(c[i]);
                    T lo = c[i + 1];
                    c[i + 1] = z ? T(0) : c[i + 1];
                    c[i] = z ? lo : c[i];
                }
            }
        }
        // trailing zeros written by the reference's compaction are +0
#pragma unroll
        for (int i = 0; i < K; ++i) c[i] = is_zero<kInt>(c[i]) ? T(0) : c[i];
        // The reference assigns (s, e) only when they differ from (c[i], c[i+1]);
        // assigning always is the same: with no difference they are equal
        // numerically and not NaN, and no -0 is present on either side (the
        // compaction above leaves nonzeros and +0; fl(a + b) is -0 only for a =
        // b = -0, and fl(b - t) only for b = -0), so they are equal bitwise.
        bool changed = false;
#pragma unroll
        for (int i = K - 2; i >= 0; --i) {
            T s, e;
            fast_two_sum(c[i], c[i + 1], s, e);
            changed = changed || !same<kInt>(s, c[i]) || !same<kInt>(e, c[i + 1]);
            c[i] = s;
            c[i + 1] = e;
        }
        if (!changed) break;
    }
#pragma unroll
    for (int i = 0; i < K; ++i) c[i] = is_zero<kInt>(c[i]) ? T(0) : c[i];
}

// multifloat.hpp:46-63 over N terms (zero terms are transparent)
template <int K, int N, bool kInt = false, typename T>
OZK_HD void extract_components(const T* t, T* out) {
#pragma unroll
    for (int q = 0; q < K; ++q) out[q] = T(0);
    T acc = t[0];
    int j = 0;
#pragma unroll
    for (int i = 1; i < N; ++i) {
        if (j < K) {
            T hi, lo;
            two_sum(acc, t[i], hi, lo);
            if (is_zero<kInt>(lo)) {
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

// extract_components<K, K+1> when t[1] is the exact rounding error of
// t[0] = fl(a + b) (vec_sum's last two_sum): the first step two_sum(t[0], t[1])
// then returns hi = t[0] (t[0] + t[1] = a + b exactly, and fl(a + b) = t[0]),
// lo = t[1] (two_sum is error-free without overflow), so it reduces to a zero
// test.  The one signed-zero exception, t[0] = -0 with t[1] = +0 (hi would be
// +0), needs every term to be -0; callers exclude it (kw_add_fast's guard).
template <int K, bool kInt, typename T>
OZK_HD void extract_after_vec_sum(const T* t, T* out) {
#pragma unroll
    for (int q = 0; q < K; ++q) out[q] = T(0);
    const bool emit = !is_zero<kInt>(t[1]);
    out[0] = emit ? t[0] : T(0);
    T acc = emit ? t[1] : t[0];
    int j = emit ? 1 : 0;
#pragma unroll
    for (int i = 2; i <= K; ++i) {
        // j <= i - 1 < K: the reference's `if (j < K)` always holds here
        T hi, lo;
        two_sum(acc, t[i], hi, lo);
        if (is_zero<kInt>(lo)) {
            acc = hi;
        } else {
#pragma unroll
            for (int q = 0; q < K; ++q) out[q] = (j == q) ? hi : out[q];
            ++j;
            acc = lo;
        }
    }
#pragma unroll
    for (int q = 0; q < K; ++q) out[q] = (j == q) ? acc : out[q];
}

// Guard of the K >= 3 fast path: every word finite with |w| < 2^1000 (2^120
// for binary32) -- so sum_ordered's finiteness probe cannot fail and no sweep
// can overflow -- and not all words zero.  Integer operations only.

template <int K, typename T>
OZK_HD bool kw_fast_ok(const T* x, T y) {
    constexpr uint32_t kSafeHi = (uint32_t)(Bits<T>::kSafe >> (sizeof(T) == 8 ? 32 : 0));
    uint32_t mx = hi_word(y) & 0x7fffffffu, any = mx | lo_word(y);
#pragma unroll
    for (int i = 0; i < K; ++i) {
        const uint32_t a = hi_word(x[i]) & 0x7fffffffu;
        mx = a > mx ? a : mx;
        any |= a | lo_word(x[i]);
    }
    return mx < kSafeHi && any != 0;
}

// MultiFloat<K> + word (multifloat.hpp:203-213); x is updated in place.  T is
// the word type: double for DD/TD/QD, float for TS (which uses the generic
// K >= 3 branch with binary32 words, see oracle/ozk_oracle.c).
// kLead (K >= 3): the caller guarantees that y precedes x[1] in merge order
// whenever x[0] precedes y, so merge_components places y right before or
// right after x[0] and only that one comparison is made (kw_sub_piece).
template <int K, bool kInt, typename T, bool kFast = false, bool kLead = false>
OZK_HD void kw_add_impl(T* x, T y) {
    if constexpr (K == 2) {
        T s, e;
        two_sum(x[0], y, s, e);
        T v = rn_add(x[1], e);
        T fs, fe;
        fast_two_sum(s, v, fs, fe);
        // from_pair (multifloat.hpp:384-392)
        if (!is_finite(fs)) {
            x[0] = fs;
            x[1] = T(0);
            return;
        }
        T ps, pe;
        fast_two_sum(fs, fe, ps, pe);
        x[0] = is_zero<kInt>(ps) ? T(0) : ps;
        x[1] = (is_zero<kInt>(pe) || is_zero<kInt>(ps)) ? T(0) : pe;
    } else {
        // merge_components(x, K, &y, 1): y goes before the first x[i] that
        // does not precede it
        T m[K + 1];
        if constexpr (kLead) {
            const bool x0_first = merge_before<kInt>(x[0], y);
            m[0] = x0_first ? x[0] : y;
            m[1] = x0_first ? y : x[0];
#pragma unroll
            for (int i = 2; i <= K; ++i) m[i] = x[i - 1];
        } else {
            bool placed = false;
#pragma unroll
            for (int i = 0; i <= K; ++i) {
                bool take_x = !placed && i < K && merge_before<kInt>(x[i < K ? i : 0], y);
                T prev = x[i > 0 ? i - 1 : 0];
                T cur = x[i < K ? i : K - 1];
                m[i] = placed ? prev : (take_x ? cur : y);
                placed = placed || !take_x;
            }
        }
        // sum_ordered: finiteness probe over all terms (cannot fail under the
        // kw_fast_ok guard: |probe| < (K + 1) * 2^1000)
        if constexpr (!kFast) {
            T probe = T(0);
#pragma unroll
            for (int i = 0; i <= K; ++i) probe = rn_add(probe, m[i]);
            if (!is_finite(probe)) {
                non_finite<K>(probe, x);
                return;
            }
        }
        // vec_sum over all K+1 terms (zeros transparent, see header)
        T s = m[K];
#pragma unroll
        for (int i = K - 1; i >= 0; --i) {
            T hi, lo;
            two_sum(m[i], s, hi, lo);
            s = hi;
            m[i + 1] = lo;
        }
        m[0] = s;
        // from_expansion.  Its output has zeros only at the tail: every word
        // it emits before the last is a two_sum hi with lo != 0 (hi == 0
        // would make the sum exact, lo == 0), and the fast path's leading
        // t[0] is emitted only with t[1] != 0 (t[1] is t[0]'s rounding
        // error), so strict_normalize's first compaction has nothing to move.
        if constexpr (kFast) {
            extract_after_vec_sum<K, kInt>(m, x);
            strict_normalize<K, kInt, OZK_KW_TAILSKIP != 0>(x);
        } else {
            extract_components<K, K + 1, kInt>(m, x);
            strict_normalize<K, kInt>(x);
        }
        if (is_zero<kInt>(x[0]) || !is_finite(x[0])) non_finite<K>(rn_add(x[0], T(0)), x);
    }
}

#if defined(__CUDA_ARCH__)
// the complete reference sequence, out of line on the device (rarely taken);
// words passed by value so the caller's registers never go through memory
template <int K, typename T>
struct KWords {
    T w[K];
};
template <int K, typename T>
__device__ __noinline__ KWords<K, T> kw_add_full_v(KWords<K, T> v, T y) {
    kw_add_impl<K, false>(v.w, y);
    return v;
}
template <int K, typename T>
__device__ __forceinline__ void kw_add_full(T* x, T y) {
    KWords<K, T> v;
#pragma unroll
    for (int i = 0; i < K; ++i) v.w[i] = x[i];
    v = kw_add_full_v<K, T>(v, y);
#pragma unroll
    for (int i = 0; i < K; ++i) x[i] = v.w[i];
}
#else
template <int K, typename T>
inline void kw_add_full(T* x, T y) {
    kw_add_impl<K, false>(x, y);
}
#endif

// OZK_KW_FAST=0 restores the plain reference sequence everywhere (A/B builds).
#ifndef OZK_KW_FAST
#define OZK_KW_FAST 1
#endif

// kIntCmp selects the comparison flavour of the fast path (same results):
// integer ALU ops where the FP64 pipe is the contended one (the slice-GEMM
// epilogue, which shares it with the tensor cores), FP64 compares where the
// ALU pipe is (the split).
// When y only reaches the last word.  For the reference's
// operator+(MultiFloat<K>, double), K >= 3 (multifloat.hpp:203-213 ->
// :420-430 -> :405-416 -> :394-401), with
//   (i)   y != 0 and x[0..K-2] nonzero,
//   (ii)  |y| < |x[K-2]|,
//   (iii) fl(x[i] + x[i+1]) == x[i] for i < K-2 (x[0..K-2] is a strict
//         fixpoint chain),
//   (iv)  h = fl(x[K-1] + y) != 0 and fl(x[K-2] + h) == x[K-2],
// the result is x[0..K-2], h.  Proof: by (ii) merge_components places y after
// x[0..K-2] (before or after x[K-1]; both give the same below); the probe
// passes (kw_fast_ok).  If x[K-1] == 0 sum_ordered drops it and vec_sum starts
// at two_sum(x[K-2], y) = (x[K-2], y) by (iv) with h = y; otherwise vec_sum
// starts with two_sum(x[K-1], y) (either order) = (h, l), l the exact error,
// then two_sum(x[K-2], h) = (x[K-2], h) by (iv) (fl(a+b) == a makes both
// two_sum and fast_two_sum return (a, b)), and (x[i], x[i+1]) for i < K-2 by
// (iii): the terms stay x[0..K-2], h, l.  extract_components then emits x[0]
// .. x[K-2] (each following term is a nonzero exact error), and h: two_sum(h,
// l) = (h, l) as l is h's rounding error, so h is emitted with l != 0 or kept
// as the final accumulator with l == 0.  strict_normalize finds every
// adjacent pair a fixpoint by (iii)/(iv) and changes nothing.  The
// negligible case h == x[K-1] (|y| < ulp(x[K-1]) / 4) is included.  In the
// accumulation acc += C_ab at the saturating split count about half of the
// pairs (the last ~3 levels alpha+beta, |C_ab| ~ 2^(-20 (alpha+beta)) |acc|)
// fall here and cost K DADDs instead of the whole sequence.
template <bool kInt, typename T>
OZK_HD bool mag_less(T a, T b) {
    if constexpr (kInt) {
        const uint32_t ha = hi_word(a) & 0x7fffffffu, hb = hi_word(b) & 0x7fffffffu;
        return ha < hb || (ha == hb && lo_word(a) < lo_word(b));
    } else {
        return fabs_(a) < fabs_(b);
    }
}

template <int K, bool kInt, typename T>
OZK_HD bool kw_add_tail(T* x, T y) {
    bool ok = !is_zero<kInt>(y) && mag_less<kInt>(y, x[K - 2]);
#pragma unroll
    for (int i = 0; i < K - 1; ++i) ok = ok && !is_zero<kInt>(x[i]);
    if (!ok) return false;
    const T h = rn_add(x[K - 1], y);
    ok = !is_zero<kInt>(h) && same<kInt>(rn_add(x[K - 2], h), x[K - 2]);
#pragma unroll
    for (int i = 0; i + 2 < K; ++i) ok = ok && same<kInt>(rn_add(x[i], x[i + 1]), x[i]);
    if (ok) x[K - 1] = h;
    return ok;
}

// The K = 2 form (multifloat.hpp:203-207 + from_pair :384-392): with x[0], y
// nonzero, all words finite below the guard, fl(x[0] + y) == x[0] and, for
// v = fl(x[1] + y), fl(x[0] + v) == x[0], the reference returns (x[0], v):
// two_sum(x[0], y) = (x[0], y) (fl(a+b) == a gives the exact error b for
// b != 0), so its v = x[1] + e is this v; fast_two_sum(x[0], v) = (x[0], v),
// and from_pair's second fast_two_sum and zero rules leave (x[0], v) (a zero v
// is +0: x[1] + y == 0 rounds to +0).
template <bool kInt, typename T>
OZK_HD bool kw_add_tail2(T* x, T y) {
    constexpr uint32_t kSafeHi = (uint32_t)(Bits<T>::kSafe >> (sizeof(T) == 8 ? 32 : 0));
    const bool guard = (hi_word(x[0]) & 0x7fffffffu) < kSafeHi &&
                       (hi_word(x[1]) & 0x7fffffffu) < kSafeHi &&
                       (hi_word(y) & 0x7fffffffu) < kSafeHi;
    if (!guard || is_zero<kInt>(x[0]) || is_zero<kInt>(y) ||
        !same<kInt>(rn_add(x[0], y), x[0]))
        return false;
    const T v = rn_add(x[1], y);
    if (!same<kInt>(rn_add(x[0], v), x[0])) return false;
    x[1] = v;
    return true;
}

// OZK_KW_TAIL=0 disables the last-word shortcuts (A/B builds).
#ifndef OZK_KW_TAIL
#define OZK_KW_TAIL 1
#endif

// kAccum: the accumulation acc += C_ab (slice-GEMM epilogues, accumulate.cu):
// tries the last-word shortcut (kw_add_tail) first.
template <int K, typename T = double, bool kIntCmp = true, bool kAccum = false>
OZK_HD void kw_add(T* x, T y) {
#if OZK_KW_FAST
    if constexpr (K >= 3) {
        // the reference sequence minus steps that are provably no-ops on
        // guarded inputs (kw_fast_ok); anything else takes the full sequence
        if (kw_fast_ok<K>(x, y)) {
            if constexpr (kAccum && OZK_KW_TAIL)
                if (kw_add_tail<K, kIntCmp>(x, y)) return;
            kw_add_impl<K, kIntCmp, T, true>(x, y);
        } else {
            kw_add_full<K>(x, y);
        }
        return;
    }
#endif
    if constexpr (K == 2 && kAccum && OZK_KW_TAIL)
        if (kw_add_tail2<kIntCmp>(x, y)) return;
    kw_add_impl<K, false>(x, y);
}

// ---- the split's residual update ---------------------------------------------
//
// w -= x  ==  w + (-x)  (multifloat.hpp:304 -> :203-213) where x is the piece
// shift_extract(w[0], tau) = fl(fl(w[0] + tau) - tau) (ozaki.hpp:53-56), tau =
// 2^(e + sigma) with |w[0]| <= 2^e < tau, e + sigma below the shift guard.
//
// K = 2.  r0 = w[0] - x is exact and two_sum(w[0], -x) = (r0, +0): t =
// fl(w[0] + tau) lies in [tau/2, 3tau/2], so x = fl(t - tau) = t - tau
// (Sterbenz) and r0 = (w[0] + tau) - t is the rounding error of an addition,
// which is representable; two_sum then computes bb = fl(r0 - w[0]) = -x
// exactly and e = fl((w[0] - fl(r0 + x)) + (-x + x)) = +0.  So the reference's
// first two_sum is one subtraction; the rest is its sequence.
//
// K >= 3.  The merge (merge_components, :420-430) puts -x right before or right
// after w[0] whenever |w[1]| < |x| or w[0] does not precede -x: for a
// canonical residual always (x != 0 is w[0] rounded to a grid G >= ulp(w[0]),
// and |w[1]| <= ulp(w[0]) / 2 < G <= |x| when w[0] comes first), so one
// comparison places it (kw_add_impl kLead).  A non-canonical first-pass input
// (MultiFloat::from_components_unchecked, :147-151) can break that; it takes
// the generic merge, out of line so the common path stays compact.
// tests/test_kword_host.py checks both against the compiled reference.
template <int K, bool kInt, typename T>
OZK_HD void kw_add_general(T* x, T y);

template <int K, bool kInt, typename T>
OZK_HD void kw_sub_piece(T* w, T x) {
    const T y = -x;
    if constexpr (K == 2) {
        const T s = rn_sub(w[0], x);        // two_sum(w[0], y) = (s, +0)
        const T v = rn_add(w[1], T(0));
        T fs, fe;
        fast_two_sum(s, v, fs, fe);
        if (!is_finite(fs)) {               // from_pair (:384-392)
            w[0] = fs;
            w[1] = T(0);
            return;
        }
        T ps, pe;
        fast_two_sum(fs, fe, ps, pe);
        w[0] = is_zero<false>(ps) ? T(0) : ps;
        w[1] = (is_zero<false>(pe) || is_zero<false>(ps)) ? T(0) : pe;
    } else {
        if (!kw_fast_ok<K>(w, y)) {
            kw_add_full<K>(w, y);
        } else if (fabs_(w[1]) < fabs_(y) || !merge_before<kInt>(w[0], y)) {
            kw_add_impl<K, kInt, T, true, true>(w, y);
        } else {
            kw_add_general<K, kInt>(w, y);
        }
    }
}

// the generic-merge update, out of line on the device (rarely taken)
#if defined(__CUDA_ARCH__)
template <int K, bool kInt, typename T>
__device__ __noinline__ KWords<K, T> kw_add_general_v(KWords<K, T> v, T y) {
    kw_add_impl<K, kInt, T, true>(v.w, y);
    return v;
}
#endif
template <int K, bool kInt, typename T>
OZK_HD void kw_add_general(T* x, T y) {
#if defined(__CUDA_ARCH__)
    KWords<K, T> v;
#pragma unroll
    for (int i = 0; i < K; ++i) v.w[i] = x[i];
    v = kw_add_general_v<K, kInt, T>(v, y);
#pragma unroll
    for (int i = 0; i < K; ++i) x[i] = v.w[i];
#else
    kw_add_impl<K, kInt, T, true>(x, y);
#endif
}

// -MultiFloat<K> (multifloat.hpp:178-182): zero words stay +0.
template <int K, typename T>
OZK_HD void kw_neg(const T* y, T* r) {
#pragma unroll
    for (int i = 0; i < K; ++i) r[i] = y[i] == T(0) ? T(0) : -y[i];
}

// MultiFloat<K> + MultiFloat<K> (multifloat.hpp:184-199); x is updated in place.
//   K = 2: accurate double-word addition (two TwoSums, two FastTwoSums, from_pair)
//   K >= 3: merge_components(x, K, y, K) -> sum_ordered(m, 2K)
// The static merge replays the reference's two-pointer merge with predicated
// selects; sum_ordered runs over all 2K terms (zero terms transparent, see
// the header comment).
template <int K, typename T = double>
OZK_HD void kw_add_kw(T* x, const T* y) {
    if constexpr (K == 2) {
        T ss, se, ts, te;
        two_sum(x[0], y[0], ss, se);
        two_sum(x[1], y[1], ts, te);
        const T c = rn_add(se, ts);
        T vs, ve;
        fast_two_sum(ss, c, vs, ve);
        const T w = rn_add(te, ve);
        T fs, fe;
        fast_two_sum(vs, w, fs, fe);
        if (!is_finite(fs)) {
            x[0] = fs;
            x[1] = T(0);
            return;
        }
        T ps, pe;
        fast_two_sum(fs, fe, ps, pe);
        x[0] = ps == T(0) ? T(0) : ps;
        x[1] = (pe == T(0) || ps == T(0)) ? T(0) : pe;
    } else {
        T m[2 * K];
        int i = 0, j = 0;
#pragma unroll
        for (int k = 0; k < 2 * K; ++k) {
            T xi = x[0], yj = y[0];
#pragma unroll
            for (int q = 1; q < K; ++q) {
                xi = (i == q) ? x[q] : xi;
                yj = (j == q) ? y[q] : yj;
            }
            const bool take_x = (i < K) && (j >= K || merge_before(xi, yj));
            m[k] = take_x ? xi : yj;
            i += take_x ? 1 : 0;
            j += take_x ? 0 : 1;
        }
        T probe = T(0);
#pragma unroll
        for (int k = 0; k < 2 * K; ++k) probe = rn_add(probe, m[k]);
        if (!is_finite(probe)) {
            non_finite<K>(probe, x);
            return;
        }
        T s = m[2 * K - 1];
#pragma unroll
        for (int k = 2 * K - 2; k >= 0; --k) {
            T hi, lo;
            two_sum(m[k], s, hi, lo);
            s = hi;
            m[k + 1] = lo;
        }
        m[0] = s;
        extract_components<K, 2 * K>(m, x);
        strict_normalize<K>(x);
        if (x[0] == T(0) || !is_finite(x[0])) non_finite<K>(rn_add(x[0], T(0)), x);
    }
}

// ---- MultiFloat<K> x MultiFloat<K> (multifloat.hpp:218-239), for the direct
// K-word GEMM (gemm.hpp:15-31, csrc/direct.cu) -------------------------------

// two_prod with a hardware FMA (eft.hpp:60-64; the reference is built with
// -mfma, so MPMAT_HAVE_HW_FMA selects this variant, eft.hpp:75-85)
template <typename T>
OZK_HD void two_prod(T a, T b, T& p, T& e) {
#if defined(__CUDA_ARCH__)
    if constexpr (sizeof(T) == 8) {
        p = __dmul_rn(a, b);
        e = __fma_rn(a, b, -p);
    } else {
        p = __fmul_rn(a, b);
        e = __fmaf_rn(a, b, -p);
    }
#else
    p = a * b;
    e = std::fma(a, b, -p);
#endif
}
template <typename T>
OZK_HD T rn_mul(T a, T b) {
#if defined(__CUDA_ARCH__)
    if constexpr (sizeof(T) == 8) return __dmul_rn(a, b);
    else return __fmul_rn(a, b);
#else
    return a * b;
#endif
}

// from_pair (multifloat.hpp:384-392) on (s, e)
template <typename T>
OZK_HD void from_pair(T s, T e, T* x) {
    if (!is_finite(s)) {
        x[0] = s;
        x[1] = T(0);
        return;
    }
    T ps, pe;
    fast_two_sum(s, e, ps, pe);
    x[0] = ps == T(0) ? T(0) : ps;
    x[1] = (pe == T(0) || ps == T(0)) ? T(0) : pe;
}

// sum_ordered(t, N) (multifloat.hpp:405-416) -> x.  The zero compaction is
// skipped: zero terms are transparent to vec_sum and extraction (header note).
template <int K, int N, typename T>
OZK_HD void sum_ordered_n(T* t, T* x) {
    T probe = T(0);
#pragma unroll
    for (int i = 0; i < N; ++i) probe = rn_add(probe, t[i]);
    if (!is_finite(probe)) {
        non_finite<K>(probe, x);
        return;
    }
    T s = t[N - 1];
#pragma unroll
    for (int i = N - 2; i >= 0; --i) {
        T hi, lo;
        two_sum(t[i], s, hi, lo);
        s = hi;
        t[i + 1] = lo;
    }
    t[0] = s;
    extract_components<K, N>(t, x);
    strict_normalize<K>(x);
    if (x[0] == T(0) || !is_finite(x[0])) non_finite<K>(rn_add(x[0], T(0)), x);
}

// canonical_order (multifloat.hpp:68-81) as a fixed odd-even transposition
// network: the order "|a| > |b|, ties by increasing bit pattern" is a strict
// total order on distinct bit patterns, so every correct sort yields the
// insertion sort's sequence (finite inputs; NaN terms end in a non-finite
// result either way through the probe).
template <typename T>
OZK_HD bool after(T a, T b) {  // a must come after b
    const T aa = fabs_(a), ab = fabs_(b);
    if (aa != ab) return aa < ab;
    return fbits(a) > fbits(b);
}
template <int N, typename T>
OZK_HD void canonical_order_n(T* t) {
#pragma unroll
    for (int round = 0; round < N; ++round) {
#pragma unroll
        for (int i = round & 1; i + 1 < N; i += 2) {
            const bool sw = after(t[i], t[i + 1]);
            const T lo = t[i + 1];
            t[i + 1] = sw ? t[i] : lo;
            t[i] = sw ? lo : t[i];
        }
    }
}

template <int K, typename T = double>
OZK_HD void kw_mul_kw(const T* x, const T* y, T* r) {
    if constexpr (K == 2) {
        T cp, ce;
        two_prod(x[0], y[0], cp, ce);
        T cs, cerr;
        two_sum(rn_mul(x[0], y[1]), rn_mul(x[1], y[0]), cs, cerr);
        const T tail = rn_add(ce, rn_add(cs, rn_add(rn_mul(x[1], y[1]), cerr)));
        T fs, fe;
        fast_two_sum(cp, tail, fs, fe);
        from_pair(fs, fe, r);
    } else {
        constexpr int N = K * (K + 1) + K - 1;
        T t[N];
        int n = 0;
#pragma unroll
        for (int i = 0; i < K; ++i) {
#pragma unroll
            for (int j = 0; j + i < K; ++j) {
                two_prod(x[i], y[j], t[n], t[n + 1]);
                n += 2;
            }
        }
#pragma unroll
        for (int i = 1; i < K; ++i) t[n++] = rn_mul(x[i], y[K - i]);
        canonical_order_n<N>(t);
        sum_ordered_n<K, N>(t, r);
    }
}

} // namespace ozk
