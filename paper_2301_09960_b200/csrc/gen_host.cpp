// gen_host.cpp -- the reference's benchmark input generator on the host,
// bit-identical to gen_matrix_eq1<K> (proj/include/mpmat/gen.hpp:20-34), and
// parallel.
//
// The reference draws every element from ONE xoshiro256** stream
// (rng.hpp:21-54, splitmix64 seeding), row-major, with a fixed number of draws
// per element: K uniforms (the K*53-bit significand of ru, renormalised) and
// one Box-Muller normal (two uniforms), then (ru - 0.5) * exp(rn) in K-word
// arithmetic.  Because the draw count per element is fixed, element e starts
// at draw e*(K+2) of the stream.  xoshiro256**'s state update is linear over
// GF(2), so the state after s draws is T^s * state0 for a 256 x 256 bit matrix
// T; each worker thread jumps to its first element with the precomputed
// squares T^(2^i) and then generates its contiguous range sequentially.  The
// per-element arithmetic is the reference's own sequence (K-word "+ double"
// from kword.cuh, which is bit-tested against the compiled reference;
// renormalize and "* double" below, multifloat.hpp:159-171 and :242-257) and
// libm's exp/log/cos/sqrt, exactly as the reference calls them.  This file is
// compiled by g++ with -ffp-contract=off, like the reference
// (proj/CMakeLists.txt:16-20), so no product is contracted into an FMA.
//
// Used by bench.py so both arms (this library and the reference CPU path)
// time the same input bytes; tests/test_gen_host.py checks it against the
// reference generator (oracle/_ref) and its golden file.
#include <sched.h>

#include <cmath>
#include <cstdint>
#include <cstring>
#include <numbers>
#include <thread>
#include <vector>

#include "../../include/ozk.h"
#include "kword.cuh"

namespace {

// ---- xoshiro256** (rng.hpp:21-54) -------------------------------------------
struct Xoshiro {
    uint64_t s[4];
    static uint64_t rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }
    void seed(uint64_t seed) {
        uint64_t sm = seed;
        for (auto& w : s) {
            uint64_t z = (sm += 0x9e3779b97f4a7c15ull);
            z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
            z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
            w = z ^ (z >> 31);
        }
    }
    // the state transition alone (linear over GF(2))
    void advance() {
        const uint64_t t = s[1] << 17;
        s[2] ^= s[0];
        s[3] ^= s[1];
        s[1] ^= s[2];
        s[0] ^= s[3];
        s[2] ^= t;
        s[3] = rotl(s[3], 45);
    }
    uint64_t next() {
        const uint64_t r = rotl(s[1] * 5, 7) * 9;
        advance();
        return r;
    }
    double uniform() { return static_cast<double>(next() >> 11) * 0x1p-53; }
    double normal() {  // cosine branch only, two draws
        const double u1 = uniform();
        const double u2 = uniform();
        const double r = std::sqrt(-2.0 * std::log(1.0 - u1));
        return r * std::cos(2.0 * std::numbers::pi * u2);
    }
};

// 256 x 256 GF(2) matrix as 256 column vectors (column j = T applied to e_j).
struct Gf2Mat {
    uint64_t col[256][4];
};

void apply(const Gf2Mat& m, const uint64_t in[4], uint64_t out[4]) {
    uint64_t r[4] = {0, 0, 0, 0};
    for (int j = 0; j < 256; ++j)
        if ((in[j >> 6] >> (j & 63)) & 1)
            for (int w = 0; w < 4; ++w) r[w] ^= m.col[j][w];
    std::memcpy(out, r, sizeof(r));
}

// T^(2^i), i = 0..63, built once
const std::vector<Gf2Mat>& jump_powers() {
    static const std::vector<Gf2Mat> pw = [] {
        std::vector<Gf2Mat> p(64);
        for (int j = 0; j < 256; ++j) {
            Xoshiro x;
            for (int w = 0; w < 4; ++w) x.s[w] = 0;
            x.s[j >> 6] = uint64_t(1) << (j & 63);
            x.advance();
            std::memcpy(p[0].col[j], x.s, sizeof(x.s));
        }
        for (int i = 1; i < 64; ++i)
            for (int j = 0; j < 256; ++j) apply(p[i - 1], p[i - 1].col[j], p[i].col[j]);
        return p;
    }();
    return pw;
}

void jump(Xoshiro& x, uint64_t draws) {
    const auto& pw = jump_powers();
    for (int i = 0; i < 64 && draws; ++i, draws >>= 1)
        if (draws & 1) apply(pw[i], x.s, x.s);
}

// ---- K-word pieces the generator needs (multifloat.hpp) ---------------------
// vec_sum (multifloat.hpp:34-42)
template <typename T>
void vec_sum(T* t, int n) {
    T s = t[n - 1];
    for (int i = n - 2; i >= 0; --i) {
        T hi, lo;
        ozk::two_sum(t[i], s, hi, lo);
        s = hi;
        t[i + 1] = lo;
    }
    t[0] = s;
}

// from_expansion (multifloat.hpp:394-401): extract_components (:46-63) then
// strict_normalize (:363-382), non-finite/zero head rule
template <int K, typename T>
void from_expansion(const T* t, int n, T* c) {
    for (int q = 0; q < K; ++q) c[q] = T(0);
    T acc = t[0];
    int j = 0;
    bool full = false;
    for (int i = 1; i < n && !full; ++i) {
        T hi, lo;
        ozk::two_sum(acc, t[i], hi, lo);
        if (lo == T(0)) {
            acc = hi;
            continue;
        }
        c[j++] = hi;
        acc = lo;
        full = j == K;
    }
    if (!full) c[j] = acc;
    ozk::strict_normalize<K>(c);
    if (c[0] == T(0) || !std::isfinite(c[0])) {
        const T h = c[0] + T(0);
        for (int q = 0; q < K; ++q) c[q] = T(0);
        c[0] = h;
    }
}

// MultiFloat<K>::renormalize (multifloat.hpp:159-171)
template <int K, typename T>
void renormalize(const T* terms, int nterms, T* c) {
    T buf[16] = {};
    int n = 0;
    T probe = T(0);
    for (int i = 0; i < nterms; ++i) {
        probe += terms[i];
        if (terms[i] != T(0)) buf[n++] = terms[i];
    }
    for (int q = 0; q < K; ++q) c[q] = T(0);
    if (!std::isfinite(probe)) {
        c[0] = probe;
        return;
    }
    if (n == 0) return;
    vec_sum(buf, n);
    if (n > 1) vec_sum(buf, n);
    from_expansion<K>(buf, n, c);
}

// MultiFloat<K> * double (multifloat.hpp:242-257), two_prod with FMA
// (eft.hpp:60-64; the reference builds with -mfma, eft.hpp:75-85)
template <int K>
void mul_double(const double* x, double y, double* r) {
    if constexpr (K == 2) {
        const double p = x[0] * y;
        const double e = std::fma(x[0], y, -p);
        const double tail = std::fma(x[1], y, e);
        double s, f;
        ozk::fast_two_sum(p, tail, s, f);
        ozk::from_pair(s, f, r);
    } else {
        double t[2 * K];
        for (int i = 0; i < K; ++i) {
            t[2 * i] = x[i] * y;
            t[2 * i + 1] = std::fma(x[i], y, -t[2 * i]);
        }
        // canonical_order (multifloat.hpp:68-81): insertion sort, |value|
        // decreasing, ties by increasing bit pattern
        for (int i = 1; i < 2 * K; ++i) {
            const double v = t[i], av = std::fabs(v);
            int j = i - 1;
            while (j >= 0 && (std::fabs(t[j]) < av ||
                              (std::fabs(t[j]) == av && ozk::fbits(t[j]) > ozk::fbits(v)))) {
                t[j + 1] = t[j];
                --j;
            }
            t[j + 1] = v;
        }
        // sum_ordered (multifloat.hpp:405-416)
        double probe = 0.0;
        for (int i = 0; i < 2 * K; ++i) probe += t[i];
        for (int q = 0; q < K; ++q) r[q] = 0.0;
        if (!std::isfinite(probe)) {
            r[0] = probe;
            return;
        }
        double buf[2 * K];
        int m = 0;
        for (int i = 0; i < 2 * K; ++i)
            if (t[i] != 0.0) buf[m++] = t[i];
        if (m == 0) return;
        vec_sum(buf, m);
        from_expansion<K>(buf, m, r);
    }
}

// One Eq. (1) element from the stream: gen.hpp:26-31 (+ the exponent-spread
// scaling of config 5 when spread > 0: one more draw, 2^U[-spread, spread])
template <int K>
void element(Xoshiro& rng, int spread, double* out) {
    double comp[K], ru[K], t[K];
    for (int k = 0; k < K; ++k) comp[k] = std::scalbn(rng.uniform(), -53 * k);
    renormalize<K>(comp, K, ru);
    const double scale = std::exp(rng.normal());
    for (int k = 0; k < K; ++k) t[k] = ru[k];
    ozk::kw_add<K>(t, -0.5);  // ru - 0.5 == ru + (-0.5) (multifloat.hpp:215)
    mul_double<K>(t, scale, out);
    if (spread > 0) {
        const int e = (int)(rng.next() % (uint64_t)(2 * spread + 1)) - spread;
        for (int k = 0; k < K; ++k) out[k] = std::scalbn(out[k], e);
    }
}

// TS: the TD value rounded to three binary32 words by successive leading-word
// extraction in binary64, then renormalised in binary32 (the repo's TS
// definition, oracle/ozk_oracle.c ozk_oracle_gen_eq1_ts)
void to_ts(const double* c, float* o) {
    float w[3];
    const double r0 = c[0];
    w[0] = (float)r0;
    const double r1 = (r0 - (double)w[0]) + c[1];
    w[1] = (float)r1;
    const double r2 = (r1 - (double)w[1]) + c[2];
    w[2] = (float)r2;
    renormalize<3>(w, 3, o);
}

template <int K>
void gen_range(uint64_t seed, size_t e0, size_t e1, int spread, bool ts, void* out) {
    Xoshiro rng;
    rng.seed(seed);
    jump(rng, (uint64_t)e0 * (uint64_t)(K + 2 + (spread > 0 ? 1 : 0)));
    double v[K];
    for (size_t e = e0; e < e1; ++e) {
        if (ts) {
            element<K>(rng, spread, v);
            if constexpr (K == 3) to_ts(v, static_cast<float*>(out) + e * 3);
        } else {
            element<K>(rng, spread, static_cast<double*>(out) + e * K);
        }
    }
}

ozk_status gen_host(ozk_format fmt, size_t rows, size_t cols, uint64_t seed, int spread,
                    void* out, int threads) {
    if (fmt != OZK_DD && fmt != OZK_TD && fmt != OZK_QD && fmt != OZK_TS) return OZK_EPARAM;
    if (rows == 0 || cols == 0) return OZK_ESHAPE;
    if (spread < 0 || spread > 400 || !out) return OZK_EPARAM;
    const size_t count = rows * cols;
    const bool ts = fmt == OZK_TS;
    const int K = ts ? 3 : (int)fmt;
    int nt = threads;
    if (nt <= 0) {  // the CPUs this process may run on (cgroup / taskset aware)
        cpu_set_t set;
        nt = sched_getaffinity(0, sizeof(set), &set) == 0 ? CPU_COUNT(&set)
                                                          : (int)std::thread::hardware_concurrency();
    }
    if (nt < 1) nt = 1;
    if ((size_t)nt > count / 4096 + 1) nt = (int)(count / 4096 + 1);
    auto run = [&](size_t e0, size_t e1) {
        switch (K) {
        case 2: gen_range<2>(seed, e0, e1, spread, false, out); break;
        case 3: gen_range<3>(seed, e0, e1, spread, ts, out); break;
        default: gen_range<4>(seed, e0, e1, spread, false, out); break;
        }
    };
    if (nt == 1) {
        run(0, count);
        return OZK_OK;
    }
    jump_powers();  // built once, before the workers read it
    std::vector<std::thread> pool;
    for (int t = 0; t < nt; ++t)
        pool.emplace_back(run, count * t / nt, count * (t + 1) / nt);
    for (auto& th : pool) th.join();
    return OZK_OK;
}

}  // namespace

extern "C" {

ozk_status ozk_gen_eq1(ozk_format fmt, size_t rows, size_t cols, uint64_t seed, void* out,
                       int threads) {
    return gen_host(fmt, rows, cols, seed, 0, out, threads);
}

ozk_status ozk_gen_spread(ozk_format fmt, size_t rows, size_t cols, uint64_t seed, int spread,
                          void* out, int threads) {
    return gen_host(fmt, rows, cols, seed, spread, out, threads);
}

}  // extern "C"
