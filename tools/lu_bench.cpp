// lu_bench.cpp -- blocked LU (lu.hpp:95-124) timed two ways on
// the same matrix: the reference's blocked_lu with its Ozaki trailing update
// on the host cores (reference_backend(), OpenMP), and the same loop with the
// trailing update A22 -= L21 * U12 on the B200 (ozk_lu_trailing_update on the
// blocks in place: INTEGRATION.md's maintainer patch).  The panel
// factorisation and the U12 solve are the reference's own serial K-word code
// in both (lu.hpp:35-70).  Factors and pivots must be bit-identical.
//
//   tools/_build/lu_bench K n panel d      (built by __graft_entry__.build())
#include <chrono>
#include <cstdio>
#include <cstdlib>

#include "mpmat/backend.hpp"
#include "mpmat/gen.hpp"
#include "mpmat/lu.hpp"
#include "mpmat_gpu.hpp"

using namespace mpmat;
using clk = std::chrono::steady_clock;

template <int K>
LuFactors<K> blocked_lu_b200(const DenseMatrix<MultiFloat<K>>& a, std::size_t panel, int d,
                             double& panel_s, double& update_s) {
    const std::size_t n = a.rows();
    LuFactors<K> f{a, std::vector<std::size_t>(n), panel};
    auto& w = f.lu;
    double* base = gpu::words(w);
    panel_s = update_s = 0.0;
    for (std::size_t j0 = 0; j0 < n; j0 += panel) {
        const std::size_t pw = std::min(panel, n - j0);
        auto t0 = clk::now();
        detail::panel_factor(w, f.pivots, j0, pw);
        if (j0 + pw == n) {
            panel_s += std::chrono::duration<double>(clk::now() - t0).count();
            break;
        }
        detail::panel_u12(w, j0, pw);
        auto t1 = clk::now();
        panel_s += std::chrono::duration<double>(t1 - t0).count();
        const std::size_t tm = n - j0 - pw;
        gpu::throw_on(ozk_lu_trailing_update(static_cast<ozk_format>(K), tm, pw, tm,
                                             base + ((j0 + pw) * n + j0) * K, n,
                                             base + (j0 * n + j0 + pw) * K, n,
                                             base + ((j0 + pw) * n + j0 + pw) * K, n, d));
        update_s += std::chrono::duration<double>(clk::now() - t1).count();
    }
    return f;
}

template <int K>
int run(std::size_t n, std::size_t panel, int d) {
    auto a = gen_matrix_eq1<K>(n, n, 1);
    GemmChoice choice;
    choice.path = GemmPath::ozaki;
    choice.split_count = d;
    // warm the GPU path (context, pools) on a small problem
    {
        auto s = gen_matrix_eq1<K>(64, 64, 2);
        double p, u;
        (void)blocked_lu_b200(s, 32, d, p, u);
    }
    auto t0 = clk::now();
    double panel_s = 0.0, update_s = 0.0;
    auto gpu = blocked_lu_b200(a, panel, d, panel_s, update_s);
    const double t_gpu = std::chrono::duration<double>(clk::now() - t0).count();
    t0 = clk::now();
    auto ref = blocked_lu(a, panel, choice);
    const double t_ref = std::chrono::duration<double>(clk::now() - t0).count();
    const bool same = ref.lu == gpu.lu && ref.pivots == gpu.pivots;
    std::printf("{\"K\": %d, \"n\": %zu, \"panel\": %zu, \"d\": %d, \"reference_s\": %.3f, "
                "\"b200_trailing_s\": %.3f, \"b200_panel_s\": %.3f, \"b200_update_s\": %.3f, "
                "\"speedup\": %.2f, \"bit_identical\": %s}\n",
                K, n, panel, d, t_ref, t_gpu, panel_s, update_s, t_ref / t_gpu,
                same ? "true" : "false");
    return same ? 0 : 1;
}

int main(int argc, char** argv) {
    const int K = argc > 1 ? std::atoi(argv[1]) : 2;
    const std::size_t n = argc > 2 ? std::strtoull(argv[2], nullptr, 10) : 1024;
    const std::size_t panel = argc > 3 ? std::strtoull(argv[3], nullptr, 10) : 128;
    const int d = argc > 4 ? std::atoi(argv[4]) : 6;
    switch (K) {
    case 2: return run<2>(n, panel, d);
    case 3: return run<3>(n, panel, d);
    case 4: return run<4>(n, panel, d);
    default: return 2;
    }
}
