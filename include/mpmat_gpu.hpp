// mpmat_gpu.hpp -- header-only C++ drop-in for the reference mpmat hot path.
//
// Same names, signatures, argument meaning and exceptions as the reference
// (paths relative to /root/reference/proj/include/mpmat/), implemented over
// the C-ABI in ozk.h (link with libozk.so):
//
//   mpmat::gpu::ozaki_gemm<K>(a, b, d, backend, drop)   ozaki.hpp:180-183
//     (fused on the B200, or with a caller's GemmBackend called once per pair)
//   mpmat::gpu::split_matrix<K>(m, d, side)             ozaki.hpp:74-75
//   mpmat::gpu::backend()  -> GemmBackend               backend.hpp:12-20
//
// Include it after (or instead of) the reference headers: it needs
// DenseMatrix, MultiFloat, SplitSet, OzakiProfile, GemmBackend and the error
// types from the reference's own headers.  DenseMatrix<MultiFloat<K>>::data()
// is K contiguous doubles per element (multifloat.hpp:131), exactly the ABI
// layout, so no element is copied or converted at the boundary.
#pragma once

#include <chrono>
#include <cmath>
#include <cstring>
#include <string>
#include <utility>
#include <vector>

#include "mpmat/ozaki.hpp"
#include "ozk.h"

namespace mpmat::gpu {

inline void throw_on(ozk_status s) {
    if (s == OZK_OK) return;
    std::string msg = ozk_last_error();
    if (s == OZK_ESHAPE) throw shape_error(msg);
    if (s == OZK_EPARAM) throw param_error(msg);
    if (s == OZK_EIO) throw io_error(msg);
    throw error(msg);
}

template <int K>
inline const double* words(const DenseMatrix<MultiFloat<K>>& m) {
    static_assert(sizeof(MultiFloat<K>) == K * sizeof(double), "MultiFloat<K> is K doubles");
    return reinterpret_cast<const double*>(m.data());
}

template <int K>
inline double* words(DenseMatrix<MultiFloat<K>>& m) {
    return reinterpret_cast<double*>(m.data());
}

// GemmBackend on the B200 DMMA kernel (reentrant: private stream per call).
// A named functor, so ozaki_gemm can recognise it inside a GemmBackend.
struct GpuBackend {
    DenseMatrix<double> operator()(const DenseMatrix<double>& a,
                                   const DenseMatrix<double>& b) const {
        if (a.cols() != b.rows()) throw shape_error("gpu backend: inner dimensions differ");
        DenseMatrix<double> c(a.rows(), b.cols());
        throw_on(ozk_backend_gemm(a.rows(), a.cols(), b.cols(), a.data(), b.data(), c.data()));
        return c;
    }
};

inline GemmBackend backend() { return GpuBackend{}; }

template <int K>
SplitSet<K> split_matrix(const DenseMatrix<MultiFloat<K>>& m, int d, SplitSide side);

// ozaki_gemm<K> with the reference's signature and semantics (ozaki.hpp:180-249).
//  * backend empty or gpu::backend(): the whole scheme runs fused on the B200
//    (exact INT8 tcgen05 digit GEMMs where they apply, FP64 DMMA otherwise,
//    the accumulation in the GEMM epilogue).  Any conforming backend gives
//    the same C (test_ozaki.cpp:227-233), so this is the same result.
//  * any other backend: the caller's plugin forms the slice products, as the
//    reference does -- once per pair of the (pruned) triangular set, in an
//    OpenMP dynamic loop when OpenMP is on (ozaki.hpp:223-231), so a
//    counting or shuffling backend sees exactly the reference's calls.  The
//    split (both sides) and the accumulation (ozaki.hpp:235-244) run on the
//    B200.
template <int K>
std::pair<DenseMatrix<MultiFloat<K>>, OzakiProfile>
ozaki_gemm(const DenseMatrix<MultiFloat<K>>& a, const DenseMatrix<MultiFloat<K>>& b, int d,
           const GemmBackend& backend = GemmBackend{}, double drop_threshold = 0.0) {
    if (a.cols() != b.rows()) throw shape_error("ozaki_gemm: inner dimensions differ");
    if (!backend || backend.template target<GpuBackend>() != nullptr) {
        DenseMatrix<MultiFloat<K>> c(a.rows(), b.cols());
        ozk_profile p{};
        throw_on(ozk_ozaki_gemm(static_cast<ozk_format>(K), a.rows(), a.cols(), b.cols(),
                                words(a), words(b), d, drop_threshold, words(c), &p));
        OzakiProfile prof;
        prof.split_seconds = p.split_seconds;
        prof.product_seconds = p.product_seconds;
        prof.accumulate_seconds = p.accumulate_seconds;
        prof.split_count = p.split_count;
        return {std::move(c), prof};
    }
    if (d < 1) throw param_error("ozaki_gemm: split count must be >= 1");
    if (drop_threshold < 0.0) throw param_error("ozaki_gemm: negative drop threshold");
    using clock = std::chrono::steady_clock;
    OzakiProfile prof;
    prof.split_count = d;
    const auto t0 = clock::now();
    SplitSet<K> sa = gpu::split_matrix(a, d, SplitSide::rows);
    SplitSet<K> sb = gpu::split_matrix(b, d, SplitSide::cols);
    const auto t1 = clock::now();
    prof.split_seconds = std::chrono::duration<double>(t1 - t0).count();
    // slice maxima and the pair list (ozaki.hpp:194-221)
    std::vector<double> amax(static_cast<std::size_t>(d)), bmax(static_cast<std::size_t>(d));
    auto piece_max = [](const DenseMatrix<double>& p) {
        double mx = 0.0;
        for (std::size_t i = 0; i < p.size(); ++i) mx = std::fmax(mx, std::fabs(p.data()[i]));
        return mx;
    };
    for (int i = 0; i < d; ++i) {
        amax[static_cast<std::size_t>(i)] = piece_max(sa.pieces[static_cast<std::size_t>(i)]);
        bmax[static_cast<std::size_t>(i)] = piece_max(sb.pieces[static_cast<std::size_t>(i)]);
    }
    std::vector<int> pairs(2 * static_cast<std::size_t>(d) * static_cast<std::size_t>(d));
    int np = 0;
    throw_on(ozk_pair_list(d, amax.data(), bmax.data(), drop_threshold, pairs.data(), &np));
    // the caller's backend, once per pair (ozaki.hpp:223-231)
    std::vector<DenseMatrix<double>> products(static_cast<std::size_t>(np));
#ifdef _OPENMP
#pragma omp parallel for schedule(dynamic)
#endif
    for (std::ptrdiff_t p = 0; p < static_cast<std::ptrdiff_t>(np); ++p)
        products[static_cast<std::size_t>(p)] =
            backend(sa.pieces[static_cast<std::size_t>(pairs[2 * p])],
                    sb.pieces[static_cast<std::size_t>(pairs[2 * p + 1])]);
    const auto t2 = clock::now();
    prof.product_seconds = std::chrono::duration<double>(t2 - t1).count();
    DenseMatrix<MultiFloat<K>> c(a.rows(), b.cols());
    std::vector<const double*> ptrs(static_cast<std::size_t>(np));
    for (int p = 0; p < np; ++p) {
        if (products[static_cast<std::size_t>(p)].rows() != a.rows() ||
            products[static_cast<std::size_t>(p)].cols() != b.cols())
            throw shape_error("ozaki_gemm: backend returned a product of the wrong shape");
        ptrs[static_cast<std::size_t>(p)] = products[static_cast<std::size_t>(p)].data();
    }
    throw_on(ozk_accumulate_products(static_cast<ozk_format>(K), a.rows(), b.cols(), ptrs.data(),
                                     np, words(c)));
    prof.accumulate_seconds = std::chrono::duration<double>(clock::now() - t2).count();
    return {std::move(c), prof};
}

template <int K>
SplitSet<K> split_matrix(const DenseMatrix<MultiFloat<K>>& m, int d, SplitSide side) {
    SplitSet<K> out;
    out.side = side;
    out.split_count = d;
    out.inner_dim = side == SplitSide::rows ? m.cols() : m.rows();
    out.residual = DenseMatrix<MultiFloat<K>>(m.rows(), m.cols());
    const int dd = d < 1 ? 1 : d;
    std::vector<double> pieces(static_cast<std::size_t>(dd) * m.size());
    throw_on(ozk_split(static_cast<ozk_format>(K), m.rows(), m.cols(), words(m), d,
                       side == SplitSide::rows ? OZK_SIDE_ROWS : OZK_SIDE_COLS, pieces.data(),
                       words(out.residual)));
    for (int i = 0; i < d; ++i) {
        DenseMatrix<double> p(m.rows(), m.cols());
        std::memcpy(p.data(), pieces.data() + static_cast<std::size_t>(i) * m.size(),
                    m.size() * sizeof(double));
        out.pieces.push_back(std::move(p));
    }
    return out;
}

} // namespace mpmat::gpu
