// ref_shim.cpp -- C entry points over the UNMODIFIED reference mpmat hot path.
//
// TEST INFRASTRUCTURE ONLY (see oracle/ozk_oracle.c header for who may load it).
// This file contains no reference code: it #includes the reference headers
// where they lie (/root/reference/proj/include) and is linked with the
// reference's own proj/src/backend.cpp, both compiled by oracle/Makefile with
// the reference's flags (proj/CMakeLists.txt:16-20,30-31) into
// oracle/_ref/libref_oracle.so.  Parity tests and bench.py --impl reference
// call through these wrappers.
#include "mpmat/backend.hpp"
#include "mpmat/dense_matrix.hpp"
#include "mpmat/gemm.hpp"
#include "mpmat/gen.hpp"
#include "mpmat/matrix_io.hpp"
#include "mpmat/ozaki.hpp"

#include <array>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>

#ifdef _OPENMP
#include <omp.h>
#endif

using namespace mpmat;

namespace {

template <int K>
DenseMatrix<MultiFloat<K>> load(std::size_t r, std::size_t c, const double* p) {
    DenseMatrix<MultiFloat<K>> m(r, c);
    for (std::size_t i = 0; i < r * c; ++i) {
        std::array<double, K> w;
        for (int k = 0; k < K; ++k) w[k] = p[i * K + k];
        m.data()[i] = MultiFloat<K>::from_components_unchecked(w);
    }
    return m;
}

template <int K>
void store(const DenseMatrix<MultiFloat<K>>& m, double* p) {
    for (std::size_t i = 0; i < m.size(); ++i)
        for (int k = 0; k < K; ++k) p[i * K + k] = m.data()[i].component(k);
}

DenseMatrix<double> load_d(std::size_t r, std::size_t c, const double* p) {
    DenseMatrix<double> m(r, c);
    std::memcpy(m.data(), p, r * c * sizeof(double));
    return m;
}

int status_of(const std::exception& e) {
    if (dynamic_cast<const shape_error*>(&e)) return 1;
    if (dynamic_cast<const param_error*>(&e)) return 2;
    return 9;
}

template <int K>
int split_k(std::size_t rows, std::size_t cols, const double* m, int d, int side,
            double* pieces, double* residual) {
    auto mat = load<K>(rows, cols, m);
    auto s = split_matrix(mat, d, side == 0 ? SplitSide::rows : SplitSide::cols);
    for (std::size_t a = 0; a < s.pieces.size(); ++a)
        std::memcpy(pieces + a * rows * cols, s.pieces[a].data(), rows * cols * sizeof(double));
    store<K>(s.residual, residual);
    return 0;
}

template <int K>
int ozaki_k(std::size_t m, std::size_t l, std::size_t n, const double* a, const double* b, int d,
            double drop, double* c, double* prof) {
    auto A = load<K>(m, l, a);
    auto B = load<K>(l, n, b);
    auto [C, p] = ozaki_gemm(A, B, d, reference_backend(), drop);
    store<K>(C, c);
    if (prof) {
        prof[0] = p.split_seconds;
        prof[1] = p.product_seconds;
        prof[2] = p.accumulate_seconds;
        prof[3] = p.total_seconds();
    }
    return 0;
}

template <int K>
int simple_k(std::size_t m, std::size_t l, std::size_t n, const double* a, const double* b,
             double* c) {
    auto A = load<K>(m, l, a);
    auto B = load<K>(l, n, b);
    auto C = gemm_simple(A, B);
    store<K>(C, c);
    return 0;
}

template <int K>
void gen_k(std::size_t m, std::size_t n, std::uint64_t seed, double* out) {
    store<K>(gen_matrix_eq1<K>(m, n, seed), out);
}

template <int K>
void add_k(std::size_t count, const double* x, const double* y, double* out) {
    for (std::size_t i = 0; i < count; ++i) {
        std::array<double, K> w;
        for (int k = 0; k < K; ++k) w[k] = x[i * K + k];
        auto r = MultiFloat<K>::from_components_unchecked(w) + y[i];
        for (int k = 0; k < K; ++k) out[i * K + k] = r.component(k);
    }
}

template <int K>
void add_mf_k(std::size_t count, const double* x, const double* y, double* out) {
    for (std::size_t i = 0; i < count; ++i) {
        std::array<double, K> a, b;
        for (int k = 0; k < K; ++k) {
            a[k] = x[i * K + k];
            b[k] = y[i * K + k];
        }
        auto r = MultiFloat<K>::from_components_unchecked(a) +
                 MultiFloat<K>::from_components_unchecked(b);
        for (int k = 0; k < K; ++k) out[i * K + k] = r.component(k);
    }
}

template <int K>
void mul_mf_k(std::size_t count, const double* x, const double* y, double* out) {
    for (std::size_t i = 0; i < count; ++i) {
        std::array<double, K> a, b;
        for (int k = 0; k < K; ++k) {
            a[k] = x[i * K + k];
            b[k] = y[i * K + k];
        }
        auto r = MultiFloat<K>::from_components_unchecked(a) *
                 MultiFloat<K>::from_components_unchecked(b);
        for (int k = 0; k < K; ++k) out[i * K + k] = r.component(k);
    }
}

template <int K>
int lu_update_k(std::size_t tm, std::size_t pw, std::size_t tn, const double* l21,
                const double* u12, double* a22, int d) {
    auto L = load<K>(tm, pw, l21);
    auto U = load<K>(pw, tn, u12);
    auto W = load<K>(tm, tn, a22);
    auto update = ozaki_gemm(L, U, d, reference_backend()).first;
    for (std::size_t i = 0; i < tm; ++i)
        for (std::size_t j = 0; j < tn; ++j) W(i, j) -= update(i, j);
    store<K>(W, a22);
    return 0;
}

#define DISPATCH_K(K, FN, ...)                                                         \
    switch (K) {                                                                       \
    case 2: return FN<2>(__VA_ARGS__);                                                 \
    case 3: return FN<3>(__VA_ARGS__);                                                 \
    case 4: return FN<4>(__VA_ARGS__);                                                 \
    default: return 2;                                                                 \
    }

template <int K>
int mpmat_read_k(const char* path, std::size_t m, std::size_t n, double* out) {
    auto a = read_matrix_file<MultiFloat<K>>(path);
    if (a.rows() != m || a.cols() != n) return 1;
    for (std::size_t i = 0; i < m * n; ++i)
        for (int k = 0; k < K; ++k) out[i * K + k] = a.data()[i].component(k);
    return 0;
}

} // namespace

extern "C" {

int ref_set_threads(int t) {
#ifdef _OPENMP
    if (t > 0) omp_set_num_threads(t);
    return omp_get_max_threads();
#else
    (void)t;
    return 1;
#endif
}

int ref_gen_eq1(int K, std::size_t m, std::size_t n, std::uint64_t seed, double* out) {
    try {
        switch (K) {
        case 2: gen_k<2>(m, n, seed, out); return 0;
        case 3: gen_k<3>(m, n, seed, out); return 0;
        case 4: gen_k<4>(m, n, seed, out); return 0;
        default: return 2;
        }
    } catch (const std::exception& e) {
        return status_of(e);
    }
}

int ref_split(int K, std::size_t rows, std::size_t cols, const double* m, int d, int side,
              double* pieces, double* residual) {
    try {
        DISPATCH_K(K, split_k, rows, cols, m, d, side, pieces, residual);
    } catch (const std::exception& e) {
        return status_of(e);
    }
}

int ref_backend_gemm(std::size_t m, std::size_t l, std::size_t n, const double* a,
                     const double* b, double* c) {
    try {
        auto C = reference_backend_gemm(load_d(m, l, a), load_d(l, n, b));
        std::memcpy(c, C.data(), m * n * sizeof(double));
        return 0;
    } catch (const std::exception& e) {
        return status_of(e);
    }
}

int ref_ozaki_gemm(int K, std::size_t m, std::size_t l, std::size_t n, const double* a,
                   const double* b, int d, double drop, double* c, double* prof) {
    try {
        DISPATCH_K(K, ozaki_k, m, l, n, a, b, d, drop, c, prof);
    } catch (const std::exception& e) {
        return status_of(e);
    }
}

int ref_gemm_simple(int K, std::size_t m, std::size_t l, std::size_t n, const double* a,
                    const double* b, double* c) {
    try {
        DISPATCH_K(K, simple_k, m, l, n, a, b, c);
    } catch (const std::exception& e) {
        return status_of(e);
    }
}

// MultiFloat<K> + double on `count` (x_i, y_i) pairs (multifloat.hpp:203-213).
int ref_mf_add_double(int K, std::size_t count, const double* x, const double* y, double* out) {
    switch (K) {
    case 2: add_k<2>(count, x, y, out); return 0;
    case 3: add_k<3>(count, x, y, out); return 0;
    case 4: add_k<4>(count, x, y, out); return 0;
    default: return 2;
    }
}

// MultiFloat<K> + MultiFloat<K> on `count` pairs (multifloat.hpp:184-199).
int ref_mf_add_mf(int K, std::size_t count, const double* x, const double* y, double* out) {
    switch (K) {
    case 2: add_mf_k<2>(count, x, y, out); return 0;
    case 3: add_mf_k<3>(count, x, y, out); return 0;
    case 4: add_mf_k<4>(count, x, y, out); return 0;
    default: return 2;
    }
}

// MultiFloat<K> * MultiFloat<K> on `count` pairs (multifloat.hpp:218-239).
int ref_mf_mul_mf(int K, std::size_t count, const double* x, const double* y, double* out) {
    switch (K) {
    case 2: mul_mf_k<2>(count, x, y, out); return 0;
    case 3: mul_mf_k<3>(count, x, y, out); return 0;
    case 4: mul_mf_k<4>(count, x, y, out); return 0;
    default: return 2;
    }
}

// The blocked-LU trailing update exactly as the reference performs it
// (lu.hpp:104-124): update = ozaki_gemm(l21, u12, d, reference_backend()).first;
// a22(i, j) -= update(i, j).  l21: tm x pw, u12: pw x tn, a22: tm x tn (dense).
int ref_lu_update(int K, std::size_t tm, std::size_t pw, std::size_t tn, const double* l21,
                  const double* u12, double* a22, int d) {
    try {
        DISPATCH_K(K, lu_update_k, tm, pw, tn, l21, u12, a22, d);
    } catch (const std::exception& e) {
        return status_of(e);
    }
}

// MPMAT v1 files through the reference's own reader/writer (src/matrix_io.cpp).
// K = 1: DenseMatrix<double> (tag d).  Returns 0, or 4 for mpmat::io_error.
int ref_mpmat_write(const char* path, int K, std::size_t m, std::size_t n, const double* a) {
    try {
        if (K == 1) {
            write_matrix_file(path, load_d(m, n, a));
            return 0;
        }
        switch (K) {
        case 2: write_matrix_file(path, load<2>(m, n, a)); return 0;
        case 3: write_matrix_file(path, load<3>(m, n, a)); return 0;
        case 4: write_matrix_file(path, load<4>(m, n, a)); return 0;
        default: return 2;
        }
    } catch (const io_error&) {
        return 4;
    } catch (const std::exception& e) {
        return status_of(e);
    }
}

int ref_mpmat_read(const char* path, int K, std::size_t m, std::size_t n, double* out) {
    try {
        if (K == 1) {
            auto a = read_matrix_file<double>(path);
            if (a.rows() != m || a.cols() != n) return 1;
            std::memcpy(out, a.data(), m * n * sizeof(double));
            return 0;
        }
        switch (K) {
        case 2: return mpmat_read_k<2>(path, m, n, out);
        case 3: return mpmat_read_k<3>(path, m, n, out);
        case 4: return mpmat_read_k<4>(path, m, n, out);
        default: return 2;
        }
    } catch (const io_error&) {
        return 4;
    } catch (const std::exception& e) {
        return status_of(e);
    }
}

int ref_split_shift_bits(std::size_t inner) { return split_shift_bits(inner); }
int ref_exponent_ceil_log2(double x) { return exponent_ceil_log2(x); }

} // extern "C"
