// mpmat_gpu.hpp -- header-only C++ drop-in for the reference mpmat hot path.
//
// Same names, signatures, argument meaning and exceptions as the reference
// (paths relative to /root/reference/proj/include/mpmat/), implemented over
// the C-ABI in ozk.h (link with libozk.so):
//
//   mpmat::gpu::ozaki_gemm<K>(a, b, d, backend, drop)   ozaki.hpp:180-183
//   mpmat::gpu::split_matrix<K>(m, d, side)             ozaki.hpp:74-75
//   mpmat::gpu::backend()  -> GemmBackend               backend.hpp:12-20
//
// Include it after (or instead of) the reference headers: it needs
// DenseMatrix, MultiFloat, SplitSet, OzakiProfile, GemmBackend and the error
// types from the reference's own headers.  DenseMatrix<MultiFloat<K>>::data()
// is K contiguous doubles per element (multifloat.hpp:218), exactly the ABI
// layout, so no element is copied or converted at the boundary.
#pragma once

#include <cstring>
#include <string>
#include <utility>

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
inline GemmBackend backend() {
    return [](const DenseMatrix<double>& a, const DenseMatrix<double>& b) {
        if (a.cols() != b.rows()) throw shape_error("gpu backend: inner dimensions differ");
        DenseMatrix<double> c(a.rows(), b.cols());
        throw_on(ozk_backend_gemm(a.rows(), a.cols(), b.cols(), a.data(), b.data(), c.data()));
        return c;
    };
}

// ozaki_gemm<K>: the slice products run on the B200 (exact INT8 tcgen05 digit
// GEMMs where they apply, FP64 DMMA otherwise, fused with the accumulation); the
// backend argument is accepted for signature compatibility (any conforming
// backend yields the same C, test_ozaki.cpp:227-233).
template <int K>
std::pair<DenseMatrix<MultiFloat<K>>, OzakiProfile>
ozaki_gemm(const DenseMatrix<MultiFloat<K>>& a, const DenseMatrix<MultiFloat<K>>& b, int d,
           const GemmBackend& /*backend*/ = GemmBackend{}, double drop_threshold = 0.0) {
    if (a.cols() != b.rows()) throw shape_error("ozaki_gemm: inner dimensions differ");
    DenseMatrix<MultiFloat<K>> c(a.rows(), b.cols());
    ozk_profile p{};
    throw_on(ozk_ozaki_gemm(static_cast<ozk_format>(K), a.rows(), a.cols(), b.cols(), words(a),
                            words(b), d, drop_threshold, words(c), &p));
    OzakiProfile prof;
    prof.split_seconds = p.split_seconds;
    prof.product_seconds = p.product_seconds;
    prof.accumulate_seconds = p.accumulate_seconds;
    prof.split_count = p.split_count;
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
