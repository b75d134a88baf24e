// C++ drop-in check: the reference's own API surface (DenseMatrix, MultiFloat,
// gen_matrix_eq1, split_matrix, ozaki_gemm, GemmBackend) with mpmat::gpu
// substituted, against the unmodified reference on the same inputs.
// Built in the development container (needs /root/reference headers) by
// __graft_entry__.build(); run on the GPU box by tests/test_cpp_shim.py.
#include <atomic>
#include <cstdio>
#include <memory>
#include <numeric>

#include "mpmat/backend.hpp"
#include "mpmat/gen.hpp"
#include "mpmat/lu.hpp"
#include "mpmat/ozaki.hpp"
#include "mpmat_gpu.hpp"

using namespace mpmat;

static int failures = 0;

#define CHECK(cond, what)                                                  \
    do {                                                                   \
        if (!(cond)) {                                                     \
            std::printf("[FAIL] %s\n", what);                              \
            ++failures;                                                    \
        } else {                                                           \
            std::printf("[PASS] %s\n", what);                              \
        }                                                                  \
    } while (0)

// GemmBackends of the kind the reference's own tests plug in
// (test_ozaki.cpp:24-49): one summing every dot product in a seeded random
// order (any order is allowed, and on slices it must stay exact), one counting
// its calls.
GemmBackend shuffled_sum_backend(std::uint64_t seed) {
    return [seed](const DenseMatrix<double>& a, const DenseMatrix<double>& b) {
        if (a.cols() != b.rows()) throw shape_error("shuffled_sum_backend: shape");
        const std::size_t m = a.rows(), l = a.cols(), n = b.cols();
        DenseMatrix<double> c(m, n);
        Xoshiro256ss rng(seed + 7919 * m + 104729 * n + l);
        std::vector<std::size_t> idx(l);
        for (std::size_t i = 0; i < m; ++i)
            for (std::size_t j = 0; j < n; ++j) {
                std::iota(idx.begin(), idx.end(), std::size_t{0});
                for (std::size_t k = l; k > 1; --k) std::swap(idx[k - 1], idx[rng.next_u64() % k]);
                double s = 0.0;
                for (std::size_t k : idx) s += a(i, k) * b(k, j);
                c(i, j) = s;
            }
        return c;
    };
}

GemmBackend call_counting_backend(std::shared_ptr<std::atomic<int>> calls) {
    return [calls](const DenseMatrix<double>& a, const DenseMatrix<double>& b) {
        calls->fetch_add(1);
        return reference_backend_gemm(a, b);
    };
}

void check_caller_backends() {
    // a caller's backend through the drop-in: called once per pair, C bit-identical
    auto a = gen_matrix_eq1<3>(20, 20, 90);
    auto b = gen_matrix_eq1<3>(20, 20, 91);
    auto [c_ref, p_ref] = ozaki_gemm(a, b, 5, reference_backend());
    auto [c_shuf, p_shuf] = gpu::ozaki_gemm(a, b, 5, shuffled_sum_backend(12345));
    CHECK(c_ref == c_shuf, "gpu::ozaki_gemm with a shuffled-summation backend bit-identical");

    auto calls = std::make_shared<std::atomic<int>>(0);
    auto counting = call_counting_backend(calls);
    auto a3 = gen_matrix_eq1<2>(3, 3, 92);
    auto b3 = gen_matrix_eq1<2>(3, 3, 93);
    auto [c3, p3] = gpu::ozaki_gemm(a3, b3, 3, counting);
    CHECK(calls->load() == 6, "caller backend called D(D+1)/2 = 6 times for D = 3");
    CHECK(c3 == ozaki_gemm(a3, b3, 3, reference_backend()).first, "D = 3 result bit-identical");
    bool counts_ok = true, same = true;
    for (int d : {1, 2, 5, 8}) {
        calls->store(0);
        auto a5 = gen_matrix_eq1<2>(5, 4, 94);
        auto b5 = gen_matrix_eq1<2>(4, 7, 95);
        auto [cg, pg] = gpu::ozaki_gemm(a5, b5, d, counting);
        counts_ok = counts_ok && calls->load() == d * (d + 1) / 2;
        same = same && cg == ozaki_gemm(a5, b5, d, reference_backend()).first;
    }
    CHECK(counts_ok, "caller backend called D(D+1)/2 times for D = 1, 2, 5, 8");
    CHECK(same, "D = 1, 2, 5, 8 results bit-identical with a caller backend");

    // pruning: the reference and the drop-in call the backend for the same pairs
    auto aq = gen_matrix_eq1<4>(16, 24, 96);
    auto bq = gen_matrix_eq1<4>(24, 12, 97);
    auto ref_calls = std::make_shared<std::atomic<int>>(0);
    calls->store(0);
    auto [cr, pr] = ozaki_gemm(aq, bq, 10, call_counting_backend(ref_calls), 1e-40);
    auto [cg, pg] = gpu::ozaki_gemm(aq, bq, 10, counting, 1e-40);
    CHECK(ref_calls->load() == calls->load() && ref_calls->load() < 55 && cr == cg,
          "pruned pair list (drop 1e-40, QD D=10): same backend calls, C bit-identical");
    CHECK(pg.split_count == 10 && pg.product_seconds > 0.0, "caller-backend profile filled");

    // split counts above 32 (the reference only requires d >= 1)
    auto ad = gen_matrix_eq1<2>(6, 300, 98);
    auto bd = gen_matrix_eq1<2>(300, 5, 99);
    auto [c40r, p40r] = ozaki_gemm(ad, bd, 40, reference_backend());
    auto [c40g, p40g] = gpu::ozaki_gemm(ad, bd, 40);
    CHECK(c40r == c40g, "D = 40 (820 pairs: two launches) bit-identical");
}

template <int K>
void check_gemm(std::size_t m, std::size_t l, std::size_t n, int d, const char* what) {
    auto a = gen_matrix_eq1<K>(m, l, 100 + m);
    auto b = gen_matrix_eq1<K>(l, n, 200 + n);
    auto [c_ref, p_ref] = ozaki_gemm(a, b, d, reference_backend());
    auto [c_gpu, p_gpu] = gpu::ozaki_gemm(a, b, d, gpu::backend());
    CHECK(c_ref == c_gpu, what);
    CHECK(p_gpu.split_count == d, "profile split_count");
}

// The reference's blocked LU loop (lu.hpp:85-127) with its trailing update
// routed to the B200 (ozk_lu_trailing_update on the blocks in place) -- the
// maintainer patch of INTEGRATION.md, written against the reference's own
// panel kernels (detail::panel_factor / panel_u12).
template <int K>
LuFactors<K> blocked_lu_b200(const DenseMatrix<MultiFloat<K>>& a, std::size_t panel, int d) {
    const std::size_t n = a.rows();
    LuFactors<K> f{a, std::vector<std::size_t>(n), panel};
    auto& w = f.lu;
    double* base = gpu::words(w);
    for (std::size_t j0 = 0; j0 < n; j0 += panel) {
        const std::size_t pw = std::min(panel, n - j0);
        detail::panel_factor(w, f.pivots, j0, pw);
        if (j0 + pw == n) break;
        detail::panel_u12(w, j0, pw);
        const std::size_t tm = n - j0 - pw;
        gpu::throw_on(ozk_lu_trailing_update(static_cast<ozk_format>(K), tm, pw, tm,
                                             base + ((j0 + pw) * n + j0) * K, n,
                                             base + (j0 * n + j0 + pw) * K, n,
                                             base + ((j0 + pw) * n + j0 + pw) * K, n, d));
    }
    return f;
}

template <int K>
void check_lu(std::size_t n, std::size_t panel, int d, const char* what) {
    auto a = gen_matrix_eq1<K>(n, n, 300 + n);
    GemmChoice choice;
    choice.path = GemmPath::ozaki;
    choice.split_count = d;
    auto ref = blocked_lu(a, panel, choice);
    auto gpu = blocked_lu_b200(a, panel, d);
    CHECK(ref.lu == gpu.lu && ref.pivots == gpu.pivots, what);
}

int main() {
    check_caller_backends();
    check_lu<2>(96, 16, 6, "blocked LU (DD n=96, panel 16) with B200 trailing updates bit-identical");
    check_lu<4>(40, 8, 12, "blocked LU (QD n=40, panel 8) with B200 trailing updates bit-identical");
    check_gemm<2>(33, 47, 29, 6, "DD ozaki_gemm bit-identical (33x47x29, D=6)");
    check_gemm<3>(20, 64, 18, 9, "TD ozaki_gemm bit-identical (20x64x18, D=9)");
    check_gemm<4>(16, 40, 24, 12, "QD ozaki_gemm bit-identical (16x40x24, D=12)");

    auto m = gen_matrix_eq1<3>(12, 9, 74);
    for (auto side : {SplitSide::rows, SplitSide::cols}) {
        auto s_ref = split_matrix(m, 5, side);
        auto s_gpu = gpu::split_matrix(m, 5, side);
        bool same = s_ref.pieces.size() == s_gpu.pieces.size() && s_ref.residual == s_gpu.residual;
        for (std::size_t i = 0; same && i < s_ref.pieces.size(); ++i)
            same = s_ref.pieces[i] == s_gpu.pieces[i];
        CHECK(same, side == SplitSide::rows ? "split_matrix rows bit-identical"
                                            : "split_matrix cols bit-identical");
    }

    // the GPU GemmBackend plugged into the REFERENCE ozaki_gemm (backend independence)
    auto a = gen_matrix_eq1<2>(40, 40, 7);
    auto b = gen_matrix_eq1<2>(40, 40, 8);
    auto [c1, p1] = ozaki_gemm(a, b, 6, reference_backend());
    auto [c2, p2] = ozaki_gemm(a, b, 6, gpu::backend());
    CHECK(c1 == c2, "reference ozaki_gemm with gpu::backend() bit-identical");

    bool threw = false;
    try {
        (void)gpu::ozaki_gemm(a, b, 0);
    } catch (const param_error&) {
        threw = true;
    }
    CHECK(threw, "param_error for D = 0");
    threw = false;
    try {
        (void)gpu::ozaki_gemm(a, DenseMatrix<DoubleDouble>(3, 3), 2);
    } catch (const shape_error&) {
        threw = true;
    }
    CHECK(threw, "shape_error for mismatched inner dimensions");
    std::printf("%d failure(s)\n", failures);
    return failures;
}
