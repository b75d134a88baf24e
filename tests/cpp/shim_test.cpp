// C++ drop-in check: the reference's own API surface (DenseMatrix, MultiFloat,
// gen_matrix_eq1, split_matrix, ozaki_gemm, GemmBackend) with mpmat::gpu
// substituted, against the unmodified reference on the same inputs.
// Built in the development container (needs /root/reference headers) by
// __graft_entry__.build(); run on the GPU box by tests/test_cpp_shim.py.
#include <cstdio>

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
