// Host build of the device K-word library (paper_2301_09960_b200/csrc/kword.cuh),
// so its operation sequence can be checked bit-for-bit against the reference's
// MultiFloat<K>::operator+(double) on the CPU (tests/test_kword_host.py).
// Test infrastructure; compiled with -ffp-contract=off like the reference.
#include <cstddef>

#include "../../paper_2301_09960_b200/csrc/kword.cuh"

template <int K>
static void run(std::size_t n, const double* x, const double* y, double* out) {
    for (std::size_t i = 0; i < n; ++i) {
        double w[K];
        for (int k = 0; k < K; ++k) w[k] = x[i * K + k];
        ozk::kw_add<K>(w, y[i]);
        for (int k = 0; k < K; ++k) out[i * K + k] = w[k];
    }
}

template <int K>
static void run_fp(std::size_t n, const double* x, const double* y, double* out) {
    for (std::size_t i = 0; i < n; ++i) {
        double w[K];
        for (int k = 0; k < K; ++k) w[k] = x[i * K + k];
        ozk::kw_add<K, double, false>(w, y[i]);  // the split's compare flavour
        for (int k = 0; k < K; ++k) out[i * K + k] = w[k];
    }
}

template <int K, typename T>
static void run_split(std::size_t n, const T* x, const T* y, T* out) {
    for (std::size_t i = 0; i < n; ++i) {
        T w[K];
        for (int k = 0; k < K; ++k) w[k] = x[i * K + k];
        ozk::kw_sub_piece<K, false>(w, -y[i]);  // the split's w -= x, x = -y[i]
        for (int k = 0; k < K; ++k) out[i * K + k] = w[k];
    }
}

// the split's residual update on (w, -x) pairs that satisfy its precondition
extern "C" int kw_host_split_sub(int K, std::size_t n, const double* x, const double* y,
                                 double* out) {
    switch (K) {
    case 2: run_split<2>(n, x, y, out); return 0;
    case 3: run_split<3>(n, x, y, out); return 0;
    case 4: run_split<4>(n, x, y, out); return 0;
    default: return 2;
    }
}

extern "C" void kw_host_split_sub_ts(std::size_t n, const float* x, const float* y, float* out) {
    run_split<3, float>(n, x, y, out);
}

template <int K, typename T>
static void run_accum(std::size_t n, const T* x, const T* y, T* out) {
    for (std::size_t i = 0; i < n; ++i) {
        T w[K];
        for (int k = 0; k < K; ++k) w[k] = x[i * K + k];
        ozk::kw_add<K, T, true, true>(w, y[i]);  // the accumulation's flavour
        for (int k = 0; k < K; ++k) out[i * K + k] = w[k];
    }
}

// acc += y as the slice-GEMM epilogues run it (kAccum: negligible-addend exit)
extern "C" int kw_host_add_accum(int K, std::size_t n, const double* x, const double* y,
                                 double* out) {
    switch (K) {
    case 2: run_accum<2>(n, x, y, out); return 0;
    case 3: run_accum<3>(n, x, y, out); return 0;
    case 4: run_accum<4>(n, x, y, out); return 0;
    default: return 2;
    }
}

extern "C" void kw_host_add_accum_ts(std::size_t n, const float* x, const float* y, float* out) {
    run_accum<3, float>(n, x, y, out);
}

extern "C" int kw_host_add_fpcmp(int K, std::size_t n, const double* x, const double* y,
                                 double* out) {
    switch (K) {
    case 2: run_fp<2>(n, x, y, out); return 0;
    case 3: run_fp<3>(n, x, y, out); return 0;
    case 4: run_fp<4>(n, x, y, out); return 0;
    default: return 2;
    }
}

template <int K>
static void run_kw(std::size_t n, const double* x, const double* y, double* out) {
    for (std::size_t i = 0; i < n; ++i) {
        double w[K], v[K];
        for (int k = 0; k < K; ++k) {
            w[k] = x[i * K + k];
            v[k] = y[i * K + k];
        }
        ozk::kw_add_kw<K>(w, v);
        for (int k = 0; k < K; ++k) out[i * K + k] = w[k];
    }
}

// MultiFloat<K> + MultiFloat<K> on n pairs
extern "C" int kw_host_add_kw(int K, std::size_t n, const double* x, const double* y,
                              double* out) {
    switch (K) {
    case 2: run_kw<2>(n, x, y, out); return 0;
    case 3: run_kw<3>(n, x, y, out); return 0;
    case 4: run_kw<4>(n, x, y, out); return 0;
    default: return 2;
    }
}

template <int K>
static void run_mul(std::size_t n, const double* x, const double* y, double* out) {
    for (std::size_t i = 0; i < n; ++i) {
        double w[K], v[K], r[K];
        for (int k = 0; k < K; ++k) {
            w[k] = x[i * K + k];
            v[k] = y[i * K + k];
        }
        ozk::kw_mul_kw<K>(w, v, r);
        for (int k = 0; k < K; ++k) out[i * K + k] = r[k];
    }
}

// MultiFloat<K> * MultiFloat<K> on n pairs (the direct GEMM's multiply)
extern "C" int kw_host_mul_kw(int K, std::size_t n, const double* x, const double* y,
                              double* out) {
    switch (K) {
    case 2: run_mul<2>(n, x, y, out); return 0;
    case 3: run_mul<3>(n, x, y, out); return 0;
    case 4: run_mul<4>(n, x, y, out); return 0;
    default: return 2;
    }
}

extern "C" void kw_host_add_ts(std::size_t n, const float* x, const float* y, float* out) {
    for (std::size_t i = 0; i < n; ++i) {
        float w[3] = {x[3 * i], x[3 * i + 1], x[3 * i + 2]};
        ozk::kw_add<3, float>(w, y[i]);
        for (int k = 0; k < 3; ++k) out[3 * i + k] = w[k];
    }
}

template <int K>
static void run_int(std::size_t n, const double* x, const double* y, double* out) {
    for (std::size_t i = 0; i < n; ++i) {
        double w[K];
        for (int k = 0; k < K; ++k) w[k] = x[i * K + k];
        ozk::kw_add_impl<K, true>(w, y[i]);
        for (int k = 0; k < K; ++k) out[i * K + k] = w[k];
    }
}

// the integer-comparison variant the device takes for finite words < 2^1000
extern "C" int kw_host_add_int(int K, std::size_t n, const double* x, const double* y,
                               double* out) {
    switch (K) {
    case 2: run_int<2>(n, x, y, out); return 0;
    case 3: run_int<3>(n, x, y, out); return 0;
    case 4: run_int<4>(n, x, y, out); return 0;
    default: return 2;
    }
}

extern "C" int kw_host_add(int K, std::size_t n, const double* x, const double* y, double* out) {
    switch (K) {
    case 2: run<2>(n, x, y, out); return 0;
    case 3: run<3>(n, x, y, out); return 0;
    case 4: run<4>(n, x, y, out); return 0;
    default: return 2;
    }
}
