"""GPU parity: the CUDA path vs the reference CPU implementation, through the C-ABI.

Tier T1 (bit-exact): slices + residual of split_matrix, every slice product
C_ab, and the final K-word C of ozaki_gemm, against oracle/_ref (the reference
compiled in place) or, when that was not built, the C restatement.  Cases
follow proj/tests/test_ozaki.cpp and acceptance.cpp criteria 3/4/8.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def bits(x):
    return np.ascontiguousarray(x).view(np.uint64)


def assert_bitwise(got, want, what):
    g, w = bits(got), bits(want)
    if not np.array_equal(g, w):
        bad = np.flatnonzero(g.reshape(-1) != w.reshape(-1))
        i = bad[0]
        raise AssertionError(f"{what}: {len(bad)} of {g.size} words differ; first at {i}: "
                             f"got {np.ascontiguousarray(got).reshape(-1)[i].hex()} "
                             f"want {np.ascontiguousarray(want).reshape(-1)[i].hex()}")


SPLIT_CASES = [
    # K, rows, cols, d, side
    (2, 16, 16, 4, 0), (2, 16, 16, 4, 1), (3, 12, 9, 5, 1), (3, 9, 12, 5, 0),
    (4, 33, 17, 7, 0), (4, 17, 33, 7, 1), (2, 6, 4, 1, 0), (3, 5, 7, 1, 1),
    (2, 300, 257, 6, 0), (2, 257, 300, 6, 1), (4, 130, 129, 12, 1), (3, 1, 1, 3, 0),
    (2, 1, 513, 3, 0), (2, 513, 1, 3, 1),
]


@pytest.mark.parametrize("K,rows,cols,d,side", SPLIT_CASES)
def test_split_bitexact(ozk, cpu, K, rows, cols, d, side):
    m = cpu.gen_eq1(K, rows, cols, 70 + rows + cols + K)
    want_p, want_r = cpu.split(K, m, d, side)
    s = ozk.split_matrix(m, d, ozk.SplitSide(side))
    assert len(s.pieces) == d
    assert_bitwise(np.stack(s.pieces), want_p, "pieces")
    assert_bitwise(s.residual, want_r, "residual")


def test_split_zero_rows_and_cols(ozk, cpu):
    # test_ozaki.cpp:161-173: zero rows/cols are skipped without log2(0)
    m = cpu.gen_eq1(2, 6, 6, 71)
    m[2, :, :] = 0.0
    m[:, 4, :] = 0.0
    for side in (0, 1):
        want_p, want_r = cpu.split(2, m, 3, side)
        s = ozk.split_matrix(m, 3, ozk.SplitSide(side))
        assert_bitwise(np.stack(s.pieces), want_p, "pieces")
        assert_bitwise(s.residual, want_r, "residual")
    z = np.zeros((4, 5, 2))
    for d in (1, 3):
        s = ozk.split_matrix(z, d, ozk.SplitSide.rows)
        assert all((p == 0).all() for p in s.pieces)


def test_split_skipped_rows_keep_their_residual(ozk, cpu):
    # A row whose leading words are all zero is skipped on every pass
    # (ozaki.hpp:105-107) and keeps its input as the residual, tail words
    # included.  The row split reads the input in pass 0 instead of copying it
    # in sweep 0, so the skipped branch writes the residual itself: dirty the
    # device pool first so a missing write shows up as stale words.
    big = cpu.gen_eq1(3, 40, 40, 73)
    ozk.split_matrix(big, 4, ozk.SplitSide.rows)
    m = cpu.gen_eq1(3, 7, 9, 74)
    m[3, :, 0] = 0.0          # leading words zero, tails kept (not renormalised)
    m[5, :, :] = 0.0
    for d in (1, 2, 5):
        for side in (0, 1):
            want_p, want_r = cpu.split(3, m, d, side)
            s = ozk.split_matrix(m, d, ozk.SplitSide(side))
            assert_bitwise(np.stack(s.pieces), want_p, f"pieces d={d} side={side}")
            assert_bitwise(s.residual, want_r, f"residual d={d} side={side}")


@pytest.mark.parametrize("K", [2, 3, 4])
def test_split_and_gemm_noncanonical_input(ozk, cpu, K):
    """Inputs that are not canonical K-word values (overlapping, unordered,
    signed-zero words: MultiFloat::from_components_unchecked, multifloat.hpp:
    147-151) go through the split's first pass as they are; slices, residual and
    C still match the reference bit for bit (kword.cuh kw_sub_piece's generic
    fallback)."""
    rng = np.random.default_rng(900 + K)
    m = rng.standard_normal((40, 300, K)) * np.exp2(rng.integers(-6, 6, (40, 300, K)))
    m[::7, :, 1] = -0.0
    m[1::5, :, K - 1] = 0.0
    for d in (1, 3, 7):
        for side in (0, 1):
            want_p, want_r = cpu.split(K, m, d, side)
            s = ozk.split_matrix(m, d, ozk.SplitSide(side))
            assert_bitwise(np.stack(s.pieces), want_p, f"pieces K={K} d={d} side={side}")
            assert_bitwise(s.residual, want_r, f"residual K={K} d={d} side={side}")
    b = rng.standard_normal((300, 24, K)) * np.exp2(rng.integers(-6, 6, (300, 24, K)))
    for d in (4, 8):
        got, _ = ozk.ozaki_gemm(m, b, d)
        assert_bitwise(got, cpu.ozaki_gemm(K, m, b, d), f"C K={K} d={d}")


def test_split_errors(ozk, cpu):
    m = cpu.gen_eq1(2, 2, 2, 72)
    with pytest.raises(ozk.param_error):
        ozk.split_matrix(m, 0, ozk.SplitSide.rows)
    bad = m.copy()
    bad[0, 0, 0] = np.inf
    with pytest.raises(ozk.param_error):
        ozk.split_matrix(bad, 2, ozk.SplitSide.rows)
    huge = m.copy()
    huge[0, 0, :] = [2.0 ** 1000, 0.0]
    with pytest.raises(ozk.param_error):
        ozk.split_matrix(huge, 2, ozk.SplitSide.rows)


def _slices(ozk, K, mat, d, side):
    import torch
    rows, cols = mat.shape[0], mat.shape[1]
    inner = cols if side == 0 else rows
    outer = rows if side == 0 else cols
    ld = ozk.lib.ozk_slice_ld(inner)
    t = torch.from_numpy(mat).cuda()
    sl = torch.zeros((d, outer, ld), dtype=torch.float64, device="cuda")
    st = ozk.lib.ozk_split_slices_device(K, rows, cols, cols, t.data_ptr(), d, side,
                                         sl.data_ptr(), outer, None,
                                         torch.cuda.current_stream().cuda_stream)
    assert st == 0, ozk.lib.ozk_last_error()
    return sl


@pytest.mark.parametrize("K,n,d", [(2, 8, 2), (2, 24, 4), (3, 32, 3), (4, 64, 5), (2, 200, 6),
                                   (4, 129, 11)])
def test_every_slice_product_exact(ozk, cpu, port, K, n, d):
    """acceptance.cpp:143-189 / test_ozaki.cpp:212-225: every C_ab is exact."""
    import ctypes

    import torch
    a = cpu.gen_eq1(K, n, n + 3, 500 + K + n)
    b = cpu.gen_eq1(K, n + 3, n - 1, 501 + K + n)
    m, l, nn = a.shape[0], a.shape[1], b.shape[1]
    sa = _slices(ozk, K, a, d, 0)
    sb = _slices(ozk, K, b, d, 1)
    pairs = [(x, y) for x in range(d) for y in range(d - x)]
    flat = (ctypes.c_int * (2 * len(pairs)))(*[v for p in pairs for v in p])
    prods = torch.empty((len(pairs), m, nn), dtype=torch.float64, device="cuda")
    st = ozk.lib.ozk_pair_products_device(m, l, nn, sa.data_ptr(), sb.data_ptr(), d, flat,
                                          len(pairs), prods.data_ptr(),
                                          torch.cuda.current_stream().cuda_stream)
    assert st == 0, ozk.lib.ozk_last_error()
    pa, _ = cpu.split(K, a, d, 0)
    pb, _ = cpu.split(K, b, d, 1)
    got = prods.cpu().numpy()
    for p, (x, y) in enumerate(pairs):
        want, inexact = port.exact_dgemm(pa[x], pb[y])
        assert inexact == 0
        assert_bitwise(got[p], want, f"C_{x}{y}")


GEMM_CASES = [
    # K, m, l, n, d
    (2, 1, 1, 1, 2), (2, 3, 3, 3, 3), (3, 3, 3, 3, 3), (2, 5, 7, 4, 3), (2, 4, 4, 4, 2),
    (2, 6, 6, 6, 4), (3, 20, 20, 20, 5), (2, 16, 16, 16, 5), (4, 17, 33, 9, 6),
    (2, 40, 40, 40, 7), (3, 40, 40, 40, 10), (4, 40, 40, 40, 13), (2, 48, 48, 48, 8),
    (2, 129, 200, 131, 6), (3, 256, 256, 256, 9), (4, 130, 300, 140, 11),
    (2, 256, 256, 256, 6), (4, 64, 8, 300, 5),
]


@pytest.mark.parametrize("K,m,l,n,d", GEMM_CASES)
def test_ozaki_gemm_bitexact(ozk, cpu, K, m, l, n, d):
    a = cpu.gen_eq1(K, m, l, 11 + m + K)
    b = cpu.gen_eq1(K, l, n, 12 + m + K)
    want = cpu.ozaki_gemm(K, a, b, d)
    got, prof = ozk.ozaki_gemm(a, b, d)
    assert_bitwise(got, want, f"C K={K} {m}x{l}x{n} D={d}")
    assert prof.split_count == d
    assert prof.pairs == d * (d + 1) // 2


def test_ozaki_gemm_golden_bench_tiny(ozk, cpu):
    """proj/tests/golden/bench_tiny.csv end to end (max_rel_err column)."""
    import csv
    import os

    import oracle.exact as ex
    path = os.path.join(os.path.dirname(__file__), "golden", "bench_tiny.csv")
    for row in csv.DictReader(open(path)):
        n, d, seed = int(row["n"]), int(row["D"]), int(row["seed"])
        a = cpu.gen_eq1(2, n, n, seed)
        b = cpu.gen_eq1(2, n, n, seed + 1)
        c, _ = ozk.ozaki_gemm(a, b, d)
        err = ex.max_rel_error(c, ex.exact_gemm(a, b))
        assert "%.17g" % err == row["max_rel_err"]


def test_drop_threshold_matches_reference(ozk, cpu):
    """test_ozaki.cpp:275-295 pruning semantics, bit-exact."""
    a = cpu.gen_eq1(2, 16, 16, 201)
    b = cpu.gen_eq1(2, 16, 16, 202)
    for drop in (0.0, 2.0 ** -60, 2.0 ** -30, 0.5, 2.0):
        want = cpu.ozaki_gemm(2, a, b, 5, drop)
        got, prof = ozk.ozaki_gemm(a, b, 5, drop_threshold=drop)
        assert_bitwise(got, want, f"drop={drop}")
    _, prof = ozk.ozaki_gemm(a, b, 5, drop_threshold=2.0 ** -60)
    assert 5 <= prof.pairs < 15


def test_oversized_d_appends_zero_slices(ozk, cpu):
    """test_ozaki.cpp:297-303."""
    a = cpu.gen_eq1(2, 8, 8, 97)
    b = cpu.gen_eq1(2, 8, 8, 98)
    c10, _ = ozk.ozaki_gemm(a, b, 10)
    c12, _ = ozk.ozaki_gemm(a, b, 12)
    assert_bitwise(c10, c12, "D=10 vs D=12")


def test_d1_within_tolerance(ozk, cpu):
    """D = 1 is the raw 53-bit image: products round, so only a tolerance applies."""
    a = cpu.gen_eq1(2, 33, 40, 5)
    b = cpu.gen_eq1(2, 40, 21, 6)
    want = cpu.ozaki_gemm(2, a, b, 1)
    got, _ = ozk.ozaki_gemm(a, b, 1)
    mag = np.abs(a[..., 0]) @ np.abs(b[..., 0])
    assert np.all(np.abs(got[..., 0] - want[..., 0]) <= 40 * 2.0 ** -53 * mag)


def test_ozaki_gemm_errors(ozk, cpu):
    a = cpu.gen_eq1(2, 1, 1, 1)
    with pytest.raises(ozk.shape_error):
        ozk.ozaki_gemm(a, cpu.gen_eq1(2, 2, 2, 1), 2)
    with pytest.raises(ozk.param_error):
        ozk.ozaki_gemm(a, a, 0)
    with pytest.raises(ozk.param_error):
        ozk.ozaki_gemm(a, a, 3, drop_threshold=-1.0)
    bad = a.copy()
    bad[0, 0, 0] = np.nan
    with pytest.raises(ozk.param_error):
        ozk.ozaki_gemm(bad, a, 2)


def test_small_exact_case(ozk):
    """test_ozaki.cpp:253-258: [3] * [4] = [12] exactly."""
    a = np.array([[[3.0, 0.0]]])
    b = np.array([[[4.0, 0.0]]])
    c, _ = ozk.ozaki_gemm(a, b, 2)
    assert c[0, 0, 0] == 12.0 and c[0, 0, 1] == 0.0


def test_backend_gemm(ozk, cpu):
    rng = np.random.default_rng(0)
    for (m, l, n) in [(1, 1, 1), (5, 7, 3), (130, 257, 129), (64, 512, 64)]:
        a = rng.standard_normal((m, l))
        b = rng.standard_normal((l, n))
        c = ozk.gpu_backend()(a, b)
        want = a @ b
        assert np.all(np.abs(c - want) <= 1e-13 * (np.abs(a) @ np.abs(b)))
    # on split pieces every order is exact: bit-identical to the reference backend
    if hasattr(cpu, "backend_gemm"):
        x = cpu.gen_eq1(2, 40, 50, 3)
        y = cpu.gen_eq1(2, 50, 30, 4)
        pa, _ = cpu.split(2, x, 3, 0)
        pb, _ = cpu.split(2, y, 3, 1)
        for i in range(3):
            assert_bitwise(ozk.gpu_backend()(pa[i], pb[2 - i]), cpu.backend_gemm(pa[i], pb[2 - i]),
                           "backend on pieces")


def test_device_tensors(ozk, cpu):
    import torch
    a = cpu.gen_eq1(3, 70, 90, 1)
    b = cpu.gen_eq1(3, 90, 50, 2)
    want = cpu.ozaki_gemm(3, a, b, 8)
    got, prof = ozk.ozaki_gemm(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda(), 8)
    assert_bitwise(got.cpu().numpy(), want, "device path")
    assert prof.product_seconds > 0


@pytest.mark.slow
@pytest.mark.parametrize("d", [2, 6, 10])
def test_config2_dd_n4096_slices_and_sampled_c(ozk, cpu, port, d):
    """BASELINE config 2: DD n=4096, D swept; slices bit-exact on both sides and
    sampled C elements bit-exact (replayed exactly as the reference does)."""
    n = 4096
    a = cpu.gen_eq1(2, n, n, 1)
    b = cpu.gen_eq1(2, n, n, 2)
    pa, _ = cpu.split(2, a, d, 0)
    pb, _ = cpu.split(2, b, d, 1)
    sa = ozk.split_matrix(a, d, ozk.SplitSide.rows)
    assert_bitwise(np.stack(sa.pieces), pa, "A slices")
    del sa
    sb = ozk.split_matrix(b, d, ozk.SplitSide.cols)
    assert_bitwise(np.stack(sb.pieces), pb, "B slices")
    del sb
    c, prof = ozk.ozaki_gemm(a, b, d)
    rng = np.random.default_rng(d)
    ii = rng.integers(0, n, 64)
    jj = rng.integers(0, n, 64)
    pairs = np.array([(x, y) for x in range(d) for y in range(d - x)], dtype=np.int32)
    want, inexact = port.replay_elements(2, pa, pb, pairs, ii, jj)
    assert inexact == 0
    assert_bitwise(c[ii, jj], want, "sampled C")


@pytest.mark.parametrize("K,m,l,n,d,world", [(2, 300, 257, 390, 6, 3), (3, 129, 140, 256, 9, 2),
                                             (4, 64, 96, 130, 12, 4)])
def test_sharded_layout_single_gpu(ozk, cpu, K, m, l, n, d, world):
    """The sharded data path on one GPU: each emulated rank splits its B column
    block in place (ld = n) into the all-gather layout [W][D][ncb][ld], splits
    its A row block, and runs the block-addressed fused GEMM.  Its C rows must
    equal the reference's rows bit for bit."""
    import ctypes

    import torch

    from paper_2301_09960_b200.sharded import GpuOps, ShardPlan, triangular_pairs
    a = cpu.gen_eq1(K, m, l, 41)
    b = cpu.gen_eq1(K, l, n, 42)
    want = cpu.ozaki_gemm(K, a, b, d)
    A = torch.from_numpy(a).cuda()
    B = torch.from_numpy(b).cuda()
    ops = GpuOps()
    plans = [ShardPlan(K, m, l, n, d, r, world) for r in range(world)]
    p0 = plans[0]
    sb_all = ops.zeros((world, d, p0.ncb, p0.ld))
    for p in plans:
        if p.c1 > p.c0:
            ops.split(K, B[:, p.c0:p.c1], l, p.c1 - p.c0, n, d, 1, sb_all[p.rank], None)
    pairs = triangular_pairs(d)
    for p in plans:
        sa = ops.zeros((d, p.rows_local, p.ld))
        ops.split(K, A[p.r0:p.r1], p.rows_local, l, l, d, 0, sa, None)
        c = ops.zeros((p.rows_local, n, K))
        ops.gemm(p, sa, sb_all, pairs, c)
        assert_bitwise(c.cpu().numpy(), want[p.r0:p.r1], f"rank {p.rank} rows")


@pytest.mark.parametrize("K,m,l,n,d,world", [(2, 300, 600, 390, 6, 3), (3, 129, 1030, 256, 9, 2),
                                             (4, 64, 700, 130, 12, 4), (2, 50, 4100, 70, 7, 8)])
def test_sharded_digits_single_gpu(ozk, cpu, K, m, l, n, d, world):
    """The sharded INT8-engine data path on one GPU: each emulated rank splits
    its B column block in place into digit planes [D][nd][ncb][ld8] + exponents
    (asynchronous entry points, data-error flags checked at the end), the
    per-plane all-gathers place rank r's block at rows r*ncb of every
    [D][nd][W*ncb][ld8] plane exactly as ShardedOzaki's do, and every rank's
    digit-plane GEMM gives the reference's C rows bit for bit."""
    import torch

    from paper_2301_09960_b200.sharded import GpuOps, ShardPlan, triangular_pairs
    a = cpu.gen_eq1(K, m, l, 51)
    b = cpu.gen_eq1(K, l, n, 52)
    want = cpu.ozaki_gemm(K, a, b, d)
    A = torch.from_numpy(a).cuda()
    B = torch.from_numpy(b).cuda()
    ops = GpuOps()
    ops.reset_flags()
    nd, ld8 = ops.int8_layout(K, l, d)
    assert nd == 3
    plans = [ShardPlan(K, m, l, n, d, r, world) for r in range(world)]
    ncb = plans[0].ncb
    b8, gb = ops.digit_planes(d, nd, world * ncb, ld8)
    for p in plans:
        if p.c1 > p.c0:
            loc8, locg = ops.digit_planes(d, nd, ncb, ld8)
            ops.split_digits(K, B[:, p.c0:p.c1], l, p.c1 - p.c0, n, d, 1, loc8, locg, None)
            for s_ in range(d):  # what the per-plane all-gathers deliver
                for t in range(nd):
                    b8[s_, t, p.rank * ncb:(p.rank + 1) * ncb] = loc8[s_, t]
                gb[s_, p.rank * ncb:(p.rank + 1) * ncb] = locg[s_]
    pairs = triangular_pairs(d)
    for p in plans:
        a8, ga = ops.digit_planes(d, nd, p.rows_local, ld8)
        ops.split_digits(K, A[p.r0:p.r1], p.rows_local, l, l, d, 0, a8, ga, None)
        c = ops.zeros((p.rows_local, n, K))
        ops.gemm_digits(p, a8, ga, b8, gb, pairs, c)
        ops.check_flags()
        assert_bitwise(c.cpu().numpy(), want[p.r0:p.r1], f"rank {p.rank} rows")


def test_digit_entry_points_reject_inapplicable(ozk):
    """ozk_int8_digits is 0 at l <= 128 (binary64), and the digit entry points
    refuse such shapes instead of computing something else."""
    import torch

    from paper_2301_09960_b200._lib import lib
    assert lib.ozk_int8_digits(2, 128, 6) == 0
    assert lib.ozk_int8_digits(2, 129, 6) == 3
    assert lib.ozk_int8_digits(0x103, 8192, 15) == 1
    x = torch.zeros((8, 8, 2), dtype=torch.float64, device="cuda")
    dg = torch.zeros((6, 3, 8, 16), dtype=torch.int8, device="cuda")
    ex = torch.zeros((6, 8), dtype=torch.int32, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    assert lib.ozk_split_digits_device(2, 8, 8, 8, x.data_ptr(), 6, 0, dg.data_ptr(), 16, 8,
                                       ex.data_ptr(), None, st) != 0


@pytest.mark.parametrize("K,m,l,n,d", [(2, 256, 256, 256, 6), (3, 256, 256, 256, 9),
                                       (4, 256, 256, 256, 12), (2, 1000, 900, 1100, 7)])
def test_repeat_runs_race_free(ozk, cpu, K, m, l, n, d):
    """Repeated launches must all be bit-exact: catches shared-memory ring races
    (a stage released before its LDS returned was overwritten by the next TMA
    load -- found and fixed in gemm.cu; these shapes reproduced it)."""
    a = cpu.gen_eq1(K, m, l, 11 + m + K)
    b = cpu.gen_eq1(K, l, n, 12 + m + K)
    want = cpu.ozaki_gemm(K, a, b, d)
    for _ in range(3):
        got, _ = ozk.ozaki_gemm(a, b, d)
        assert_bitwise(got, want, f"K={K} {m}x{l}x{n} D={d}")


@pytest.mark.parametrize("K,m,l,n,d,spread", [(2, 48, 96, 40, 10, 40), (4, 33, 70, 20, 16, 60),
                                              (3, 64, 64, 64, 14, 100), (2, 130, 257, 129, 12, 250)])
def test_ill_conditioned_bitexact(ozk, cpu, port, K, m, l, n, d, spread):
    """BASELINE config 5 inputs (exponent spread up to 2*spread binades):
    C bit-exact vs the reference, which handles them the same way."""
    a = port.gen_spread(K, m, l, 60 + K, spread)
    b = port.gen_spread(K, l, n, 61 + K, spread)
    want = cpu.ozaki_gemm(K, a, b, d)
    got, _ = ozk.ozaki_gemm(a, b, d)
    assert_bitwise(got, want, f"spread={spread} K={K} D={d}")


@pytest.mark.parametrize("K,dmax,ulp", [(2, 12, -106), (3, 16, -159), (4, 20, -212)])
def test_accuracy_t2_bound(ozk, port, K, dmax, ulp):
    """Tier T2: at saturation |C - C_exact| <= 4 u_L (|A||B|)_ij (SURVEY §8 parity
    tiers; exact big-int oracle), including ill-conditioned (spread) inputs."""
    import oracle.exact as ex
    for spread in (0, 30):
        a = port.gen_spread(K, 20, 64, 7, spread)
        b = port.gen_spread(K, 64, 16, 8, spread)
        ref = ex.exact_gemm(a, b)
        got, _ = ozk.ozaki_gemm(a, b, dmax)
        assert ex.componentwise_ulp_error(got, a, b, ref, ulp) <= 4.0


@pytest.mark.parametrize("K,n,j0,pw,d,eng", [
    (2, 40, 8, 8, 6, "auto"), (3, 64, 16, 16, 9, "auto"), (4, 50, 10, 7, 12, "auto"),
    (2, 300, 32, 32, 6, "auto"), (2, 129, 0, 1, 4, "auto"),
    # panels wider than 128: the INT8 engine's fused subtraction (and DMMA's)
    (2, 420, 30, 160, 6, "auto"), (3, 430, 20, 200, 9, "auto"), (4, 390, 10, 150, 12, "auto"),
    (3, 430, 20, 200, 9, "dmma"),
    # 820 pairs = two launches: only the last one subtracts
    (2, 330, 0, 140, 40, "auto"), (2, 200, 0, 64, 40, "auto")])
def test_lu_trailing_update_bitexact(ozk, ref, engine, K, n, j0, pw, d, eng):
    """the blocked-LU trailing update A22 -= L21*U12
    (lu.hpp:104-124) on strided blocks of the full matrix, bit-identical to the
    reference's own ozaki_gemm + MultiFloat operator-= -- with the subtraction
    fused into the last pair's epilogue of either engine."""
    if ref is None:
        pytest.skip("oracle/_ref not built")
    engine(eng)
    w = ref.gen_eq1(K, n, n, 90 + n)
    tm = n - j0 - pw
    l21 = w[j0 + pw:, j0:j0 + pw]
    u12 = w[j0:j0 + pw, j0 + pw:]
    want = ref.lu_update(K, l21, u12, w[j0 + pw:, j0 + pw:], d)
    got = w.copy()
    ozk.lu_trailing_update(got[j0 + pw:, j0 + pw:], got[j0 + pw:, j0:j0 + pw],
                           got[j0:j0 + pw, j0 + pw:], d)
    assert_bitwise(got[j0 + pw:, j0 + pw:], want, "A22")
    assert_bitwise(got[:j0 + pw], w[:j0 + pw], "untouched rows")
    assert_bitwise(got[j0 + pw:, :j0 + pw], w[j0 + pw:, :j0 + pw], "untouched cols")
    assert tm > 0


@pytest.fixture
def engine(ozk):
    """Run a test under a chosen slice-product engine, restore auto afterwards."""
    def use(name):
        ozk.set_engine(name)
    yield use
    ozk.set_engine("auto")


I8_CASES = [
    # K, m, l, n, d  (l > 128: the exact INT8-digit engine applies)
    (2, 130, 600, 70, 6), (3, 64, 1000, 64, 9), (4, 200, 777, 130, 12), (2, 256, 2048, 256, 7),
    (2, 70, 129, 90, 6), (3, 33, 200, 47, 9), (4, 65, 256, 64, 12), (2, 40, 512, 40, 6),
    (2, 1, 513, 1, 2), (3, 300, 1024, 129, 10), (4, 129, 4096, 65, 12), (2, 64, 8192, 64, 6),
]


@pytest.mark.parametrize("K,m,l,n,d", I8_CASES)
@pytest.mark.parametrize("eng", ["int8", "dmma"])
def test_engines_bitexact(ozk, cpu, engine, eng, K, m, l, n, d):
    """Both slice-product engines (FP64 DMMA, exact INT8 digits on tcgen05)
    reproduce the reference C bit for bit."""
    engine(eng)
    a = cpu.gen_eq1(K, m, l, 5 + m + K)
    b = cpu.gen_eq1(K, l, n, 6 + m + K)
    want = cpu.ozaki_gemm(K, a, b, d)
    got, prof = ozk.ozaki_gemm(a, b, d)
    assert prof.engine == eng
    assert_bitwise(got, want, f"{eng} K={K} {m}x{l}x{n} D={d}")


@pytest.mark.parametrize("spread", [30, 200])
def test_int8_engine_ill_conditioned_and_pruning(ozk, cpu, port, engine, spread):
    engine("int8")
    a = port.gen_spread(2, 70, 700, 3, spread)
    b = port.gen_spread(2, 700, 50, 4, spread)
    for d, drop in ((10, 0.0), (10, 2.0 ** -80), (14, 0.0)):
        want = cpu.ozaki_gemm(2, a, b, d, drop)
        got, _ = ozk.ozaki_gemm(a, b, d, drop_threshold=drop)
        assert_bitwise(got, want, f"int8 spread={spread} D={d} drop={drop}")


def test_int8_engine_repeat_runs(ozk, cpu, engine):
    engine("int8")
    a = cpu.gen_eq1(4, 300, 1200, 1)
    b = cpu.gen_eq1(4, 1200, 300, 2)
    want = cpu.ozaki_gemm(4, a, b, 12)
    for _ in range(3):
        got, _ = ozk.ozaki_gemm(a, b, 12)
        assert_bitwise(got, want, "int8 repeat")


def test_int8_engine_rejects_inapplicable(ozk, engine):
    engine("int8")
    a = np.zeros((4, 100, 2))
    with pytest.raises(ozk.param_error):
        ozk.ozaki_gemm(a, np.zeros((100, 4, 2)), 6)  # l <= 128


@pytest.mark.parametrize("K,m,l,n", [(2, 33, 47, 29), (3, 20, 33, 18), (4, 16, 40, 24),
                                     (2, 64, 64, 64), (3, 17, 1, 5), (4, 1, 70, 1)])
def test_direct_gemm_bitexact(ozk, ref, K, m, l, n):
    """Direct K-word GEMM = the reference's gemm_simple<MultiFloat<K>>
    (gemm.hpp:15-31) bit for bit, host and device entry points."""
    import torch
    if ref is None:
        pytest.skip("oracle/_ref not built")
    a = ref.gen_eq1(K, m, l, 61 + K)
    b = ref.gen_eq1(K, l, n, 62 + K)
    want = ref.gemm_simple(K, a, b)
    got = ozk.gemm_simple(a, b)
    assert_bitwise(got, want, f"direct K={K} {m}x{l}x{n} (host API)")
    gd = ozk.gemm_simple(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda())
    assert_bitwise(gd.cpu().numpy(), want, f"direct K={K} {m}x{l}x{n} (device API)")


def test_direct_gemm_spread_inputs(ozk, ref, port):
    """Wide exponent range and exact cancellations inside the k loop."""
    if ref is None:
        pytest.skip("oracle/_ref not built")
    a = port.gen_spread(3, 24, 30, 5, 200)
    b = port.gen_spread(3, 30, 20, 6, 200)
    b[3] = -b[3]
    a[:, 4] = 0.0
    assert_bitwise(ozk.gemm_simple(a, b), ref.gemm_simple(3, a, b), "direct TD spread")


@pytest.mark.parametrize("K,m,l,n,d,drop", [(2, 2049, 600, 70, 6, 0.0), (3, 2048, 300, 64, 9, 2.0 ** -90),
                                            (4, 2100, 130, 40, 12, 0.0), (2, 4097, 100, 33, 6, 0.0),
                                            (3, 2048, 140, 4101, 3, 0.0), (2, 2050, 300, 4352, 4, 0.0),
                                            (4, 2048, 129, 4096, 2, 0.0), (2, 2048, 200, 4100, 3, 2.0 ** -60)])
@pytest.mark.parametrize("head", [0, 4])
def test_host_api_banded_overlap(ozk, cpu, monkeypatch, head, K, m, l, n, d, drop):
    """ozk_ozaki_gemm with host buffers at m >= 2048 runs the banded, transfer-
    overlapped schedule (B first, A + slice GEMM in 8 row bands, C copied back
    per band; drop > 0 keeps the whole-matrix A split); at n >= 4096 on the INT8
    engine B also arrives in 4 column blocks, each split as it lands, and the
    first band is multiplied block by block (ragged last block included):
    bit-identical."""
    if head:
        monkeypatch.setenv("OZK_HOST_HEAD", str(head))
    a = cpu.gen_eq1(K, m, l, 90 + K)
    b = cpu.gen_eq1(K, l, n, 91 + K)
    want = cpu.ozaki_gemm(K, a, b, d, drop)
    got, prof = ozk.ozaki_gemm(a, b, d, drop_threshold=drop)
    assert_bitwise(got, want, f"banded host K={K} {m}x{l}x{n} D={d} drop={drop}")
    assert prof.split_seconds > 0 and prof.product_seconds > 0



@pytest.mark.parametrize("K,m,l,n", [(2, 64, 8192, 48), (3, 40, 8192, 40), (4, 32, 8192, 24),
                                     (3, 50, 600, 70), (2, 33, 100, 20)])
def test_auto_split_count_matches_reference(ozk, cpu, K, m, l, n):
    """ozaki_gemm_auto = the reference's ozaki_gemm(a, b, D, backend, drop) for
    the policy's D and drop; at l = 8192 the kept pairs are those of the
    measured accuracy saturation (TD: alpha + beta <= 8 -> 45 pairs)."""
    a = cpu.gen_eq1(K, m, l, 100 + K)
    b = cpu.gen_eq1(K, l, n, 101 + K)
    got, prof, d, drop = ozk.ozaki_gemm_auto(a, b)
    want = cpu.ozaki_gemm(K, a, b, d, drop)
    assert_bitwise(got, want, f"auto K={K} l={l} D={d}")
    assert prof.pairs < d * (d + 1) // 2  # pruning removed the sub-precision pairs
    if l == 8192 and K == 3:
        assert prof.pairs == 45


@pytest.mark.parametrize("K,m,l,n,d", [(2, 70, 600, 65, 6), (3, 33, 700, 40, 9), (4, 20, 300, 31, 12)])
def test_int8_unaligned_c(ozk, cpu, engine, K, m, l, n, d):
    """C at an 8-byte (not 16-byte) aligned address: the INT8 epilogue's
    per-word access path (no 16-byte vector loads/stores), bit-identical."""
    import ctypes

    import torch
    engine("int8")
    a = cpu.gen_eq1(K, m, l, 120 + K)
    b = cpu.gen_eq1(K, l, n, 121 + K)
    want = cpu.ozaki_gemm(K, a, b, d)
    A = torch.from_numpy(a).cuda()
    B = torch.from_numpy(b).cuda()
    buf = torch.full((m * n * K + 1,), 7.0, dtype=torch.float64, device="cuda")
    C = buf[1:]  # base + 8 bytes
    assert C.data_ptr() % 16 == 8
    from paper_2301_09960_b200._lib import OzkProfile, lib
    prof = OzkProfile()
    st = lib.ozk_ozaki_gemm_device(K, m, l, n, A.data_ptr(), B.data_ptr(), d, 0.0, C.data_ptr(),
                                   torch.cuda.current_stream().cuda_stream, ctypes.byref(prof))
    assert st == 0 and prof.engine == 2
    assert_bitwise(C.view(m, n, K).cpu().numpy(), want, f"unaligned C K={K}")
    assert buf[0].item() == 7.0  # nothing written before C


@pytest.mark.parametrize("K,d,ulp,bound", [(2, 7, -106, 1.0), (3, 9, -159, 1.0), (4, 12, -212, 1.0)])
def test_accuracy_t2_large_inner_dim(ozk, port, engine, K, d, ulp, bound):
    """T2 at the headline inner dimension l = 8192 on the INT8 engine, at the
    split counts where SURVEY Appendix A measured saturation (DD 7, TD 9, QD 12):
    |C - C_exact| <= bound * u_L * (|A||B|)_ij on sampled rows (exact big-int
    oracle).  The measured saturated errors there were 0.22 / 0.128 / 0.055."""
    import oracle.exact as ex
    engine("int8")
    a = port.gen_eq1(K, 6, 8192, 17 + K)
    b = port.gen_eq1(K, 8192, 5, 27 + K)
    ref = ex.exact_gemm(a, b)
    got, prof = ozk.ozaki_gemm(a, b, d)
    assert prof.engine == "int8"
    err = ex.componentwise_ulp_error(got, a, b, ref, ulp)
    assert err <= bound, err


def test_identity_product_truncation_bounds(ozk, cpu):
    """test_ozaki.cpp:260-268: A * I is pure split truncation -- max relative
    error <= 2^-35 at D=2 and <= 2^-100 at D=6 (exact big-int oracle)."""
    import oracle.exact as ex
    m = cpu.gen_eq1(2, 10, 10, 96)
    eye = np.zeros((10, 10, 2))
    eye[np.arange(10), np.arange(10), 0] = 1.0
    ref = ex.exact_gemm(m, eye)
    c2, _ = ozk.ozaki_gemm(m, eye, 2)
    assert ex.max_rel_error(c2, ref) <= 2.0 ** -35
    c6, _ = ozk.ozaki_gemm(m, eye, 6)
    assert ex.max_rel_error(c6, ref) <= 2.0 ** -100


def test_accuracy_monotone_in_d(ozk, cpu):
    """test_ozaki.cpp:305-320: error non-increasing in D (15 % slack) from D=2,
    and <= 1e-30 at D=8 for DD n=48."""
    import oracle.exact as ex
    a = cpu.gen_eq1(2, 48, 48, 99)
    b = cpu.gen_eq1(2, 48, 48, 100)
    ref = ex.exact_gemm(a, b)
    prev = 1e300
    for d in range(2, 9):
        c, _ = ozk.ozaki_gemm(a, b, d)
        err = ex.max_rel_error(c, ref)
        assert err <= prev * 1.15, (d, err, prev)
        prev = min(prev, err)
    assert err <= 1e-30


def test_profile_accounts_for_phases(ozk, cpu):
    """test_ozaki.cpp:322-332: non-negative phase times summing to the total,
    split count and pair count reported."""
    a = cpu.gen_eq1(2, 32, 600, 101)
    b = cpu.gen_eq1(2, 600, 32, 102)
    for d in (4, 6):
        _, prof = ozk.ozaki_gemm(a, b, d)
        assert prof.split_seconds >= 0 and prof.product_seconds >= 0
        assert prof.accumulate_seconds >= 0 and prof.split_count == d
        assert prof.pairs == d * (d + 1) // 2
        assert prof.total_seconds() > 0
        fr = prof.split_fraction() + prof.product_fraction() + prof.accumulate_fraction()
        assert abs(fr - 1.0) <= 1e-12


def test_acceptance_9_ozaki_faster_than_direct(ozk):
    """acceptance.cpp:467-485 analogue on the B200: Ozaki DD D=6 at n=1024 is at
    least 1.5x faster than the direct K-word GEMM (gemm_simple) on the same
    device, both device-resident."""
    import ctypes

    import torch

    from paper_2301_09960_b200._lib import OzkProfile, lib
    n = 1024
    st = torch.cuda.current_stream().cuda_stream
    A = torch.empty((n, n, 2), dtype=torch.float64, device="cuda")
    B = torch.empty_like(A)
    C = torch.empty_like(A)
    lib.ozk_gen_eq1_device(2, n, n, 1, A.data_ptr(), st)
    lib.ozk_gen_eq1_device(2, n, n, 2, B.data_ptr(), st)
    prof = OzkProfile()

    def timed(fn):
        fn()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1)
    t_oz = timed(lambda: lib.ozk_ozaki_gemm_device(2, n, n, n, A.data_ptr(), B.data_ptr(), 6,
                                                   0.0, C.data_ptr(), st, ctypes.byref(prof)))
    t_dir = timed(lambda: lib.ozk_direct_gemm_device(2, n, n, n, A.data_ptr(), B.data_ptr(),
                                                     C.data_ptr(), st))
    assert t_dir >= 1.5 * t_oz, (t_oz, t_dir)


@pytest.mark.parametrize("K,m,l,n,d,drop,devs", [
    (3, 300, 700, 260, 9, 0.0, [0, 0]),          # INT8 engine, 2 entries on one GPU
    (2, 257, 600, 131, 6, 2.0 ** -70, [0, 0, 0]),  # pruning: host max of the slice maxima
    (4, 100, 300, 77, 12, 0.0, [0, 0, 0, 0]),     # ragged column blocks (77 = 20+20+20+17)
    (2, 90, 100, 50, 6, 0.0, [0, 0]),             # l <= 128: per-device 1-GPU path
    (3, 5, 200, 3, 4, 0.0, [0, 0, 0, 0]),         # fewer columns than devices
    (2, 64, 300, 64, 5, 0.0, [0]),                # one device
])
def test_ozaki_gemm_multi_bitexact(ozk, cpu, K, m, l, n, d, drop, devs):
    """ozk_ozaki_gemm_multi (one process, a host thread per device, B digit
    planes all-gathered by peer copies) = the reference for any device count.
    One GPU per box here, so the devices repeat; the kernels of different
    entries never wait on each other."""
    a = cpu.gen_eq1(K, m, l, 300 + K)
    b = cpu.gen_eq1(K, l, n, 301 + K)
    want = cpu.ozaki_gemm(K, a, b, d, drop)
    got, prof = ozk.ozaki_gemm_multi(a, b, d, devices=devs, drop_threshold=drop)
    assert_bitwise(got, want, f"multi K={K} {m}x{l}x{n} D={d} drop={drop} devs={devs}")


def test_ozaki_gemm_multi_ts(ozk, port):
    a = port.gen_eq1_ts(120, 1100, 7)
    b = port.gen_eq1_ts(1100, 90, 8)
    want = port.ozaki_gemm_ts(a, b, 10)
    got, _ = ozk.ozaki_gemm_multi(a, b, 10, devices=[0, 0, 0])
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))


@pytest.mark.parametrize("engine", ["auto", "dmma"])
@pytest.mark.parametrize("K,m,l,n,d", [(2, 6, 300, 5, 40), (3, 9, 64, 7, 36), (4, 5, 200, 4, 33)])
def test_split_count_above_32(ozk, cpu, engine, K, m, l, n, d):
    """The reference takes any D >= 1 (ozaki.hpp:185).  D(D+1)/2 > 528 pairs run as
    consecutive launches continuing the K-word sum; the result is unchanged."""
    a = cpu.gen_eq1(K, m, l, 600 + d)
    b = cpu.gen_eq1(K, l, n, 601 + d)
    want = cpu.ozaki_gemm(K, a, b, d)
    ozk.set_engine(engine)
    try:
        got, prof = ozk.ozaki_gemm(a, b, d)
    finally:
        ozk.set_engine("auto")
    assert prof.pairs == d * (d + 1) // 2
    assert_bitwise(got, want, f"D={d} engine={engine}")
    s = ozk.split_matrix(a, d, ozk.SplitSide.rows)
    want_p, want_r = cpu.split(K, a, d, 0)
    assert_bitwise(np.stack(s.pieces), want_p, "pieces D > 32")
    assert_bitwise(s.residual, want_r, "residual D > 32")


def test_caller_backend_called_per_pair(ozk, cpu):
    """A caller's GemmBackend (test_ozaki.cpp:24-49 counting / shuffled
    summation): called once per pair, reference order, C bit-identical."""
    calls = []

    def counting(x, y):
        calls.append((x.shape, y.shape))
        return cpu.backend_gemm(x, y)

    def shuffled(x, y):
        rng = np.random.default_rng(x.shape[0] * 131 + y.shape[1])
        order = rng.permutation(x.shape[1])
        c = np.zeros((x.shape[0], y.shape[1]))
        for k in order:
            c += np.outer(x[:, k], y[k, :])
        return c

    for K, d in ((2, 1), (2, 3), (3, 5), (4, 8)):
        a = cpu.gen_eq1(K, 5, 4, 94 + K)
        b = cpu.gen_eq1(K, 4, 7, 95 + K)
        calls.clear()
        got, prof = ozk.ozaki_gemm(a, b, d, backend=counting)
        assert len(calls) == d * (d + 1) // 2
        assert_bitwise(got, cpu.ozaki_gemm(K, a, b, d), f"counting backend K={K} D={d}")
        if d > 1:  # D = 1 products are of unsplit leading images: not exact, order-dependent
            got2, _ = ozk.ozaki_gemm(a, b, d, backend=shuffled)
            assert_bitwise(got2, got, f"shuffled backend K={K} D={d}")
    a = cpu.gen_eq1(4, 16, 24, 96)
    b = cpu.gen_eq1(4, 24, 12, 97)
    calls.clear()
    got, prof = ozk.ozaki_gemm(a, b, 10, backend=counting, drop_threshold=1e-40)
    assert 0 < len(calls) < 55 and prof.pairs == len(calls)
    assert_bitwise(got, cpu.ozaki_gemm(4, a, b, 10, drop=1e-40), "pruned, caller backend")


def test_accumulate_products_matches_reference(ozk, cpu, port):
    """ozk_accumulate_products = the reference's accumulation phase
    (ozaki.hpp:235-244) over exact slice products."""
    import ctypes
    for K, d in ((2, 6), (3, 9), (4, 12)):
        a = cpu.gen_eq1(K, 17, 40, 700 + K)
        b = cpu.gen_eq1(K, 40, 13, 701 + K)
        pa, _ = cpu.split(K, a, d, 0)
        pb, _ = cpu.split(K, b, d, 1)
        prods = []
        for x in range(d):
            for y in range(d - x):
                c, bad = port.exact_dgemm(pa[x], pb[y])
                assert bad == 0
                prods.append(c)
        ptrs = (ctypes.c_void_p * len(prods))(*[p.ctypes.data for p in prods])
        out = np.empty((17, 13, K))
        assert ozk.lib.ozk_accumulate_products(K, 17, 13, ptrs, len(prods), out.ctypes.data) == 0
        assert_bitwise(out, cpu.ozaki_gemm(K, a, b, d), f"accumulate K={K}")
    zero = np.ones((3, 4, 2))
    assert ozk.lib.ozk_accumulate_products(2, 3, 4, None, 0, zero.ctypes.data) == 0
    assert (zero == 0).all()


@pytest.mark.parametrize("n,head", [(4200, 0), (8320, 0), (8320, 4), (4200, 3)])
def test_host_api_pinned_and_pageable_agree(ozk, cpu, monkeypatch, n, head):
    """ozk_ozaki_gemm's host path with every mix of pinned (page-locked) and
    pageable caller buffers -- pageable ones are staged through pinned slots on
    worker threads (csrc/staging.cu), strided B column blocks included -- and
    with staging switched off (OZK_PAGEABLE_STAGING=0, the driver's own pageable
    copies): bit-identical C."""
    import ctypes

    import torch
    K, m, l, d = 3, 2304, 300, 4   # n = 8320: 8 ragged B column blocks
    if head:  # the 2-D head schedule: A bands interleaved with the B blocks
        monkeypatch.setenv("OZK_HOST_HEAD", str(head))
    a = cpu.gen_eq1(K, m, l, 31)
    b = cpu.gen_eq1(K, l, n, 32)
    pa, pb = torch.from_numpy(a).pin_memory(), torch.from_numpy(b).pin_memory()
    pc = torch.empty((m, n, K), dtype=torch.float64).pin_memory()
    ref_c = None
    for a_pin in (True, False):
        for b_pin in (True, False):
            for c_pin in (True, False):
                c = np.empty((m, n, K))
                st = ozk.lib.ozk_ozaki_gemm(K, m, l, n, pa.data_ptr() if a_pin else a.ctypes.data,
                                            pb.data_ptr() if b_pin else b.ctypes.data, d, 0.0,
                                            pc.data_ptr() if c_pin else c.ctypes.data, None)
                assert st == 0, ozk.lib.ozk_last_error()
                got = pc.numpy().copy() if c_pin else c
                if ref_c is None:
                    ref_c = got
                assert_bitwise(got, ref_c, f"pinned A={a_pin} B={b_pin} C={c_pin}")
    monkeypatch.setenv("OZK_PAGEABLE_STAGING", "0")
    c = np.empty((m, n, K))
    assert ozk.lib.ozk_ozaki_gemm(K, m, l, n, a.ctypes.data, b.ctypes.data, d, 0.0,
                                  c.ctypes.data, None) == 0
    assert_bitwise(c, ref_c, "staging off")
    rows = np.arange(0, m, 97)
    want = cpu.ozaki_gemm(K, np.ascontiguousarray(a[rows]), b, d)
    assert_bitwise(ref_c[rows], want, "sampled rows vs the reference")


def test_device_async_entry(ozk, cpu):
    """ozk_ozaki_gemm_device_async: several GEMMs queued back to back on one
    stream with no synchronisation in between give the synchronous entry's
    bits; data errors arrive in the device flags (A's before B's), argument
    errors in the return value."""
    import torch
    lib = ozk.lib
    st = torch.cuda.current_stream().cuda_stream
    flags = torch.full((2,), -1, dtype=torch.int32, device="cuda")
    outs, wants = [], []
    for K, m, l, n, d in ((2, 300, 257, 190, 6), (3, 64, 100, 80, 9), (4, 130, 300, 140, 11)):
        a = cpu.gen_eq1(K, m, l, 30 + K)
        b = cpu.gen_eq1(K, l, n, 31 + K)
        wants.append(cpu.ozaki_gemm(K, a, b, d))
        A, B = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
        C = torch.empty((m, n, K), dtype=torch.float64, device="cuda")
        assert lib.ozk_ozaki_gemm_device_async(K, m, l, n, A.data_ptr(), B.data_ptr(), d, 0.0,
                                               C.data_ptr(), flags.data_ptr(), st) == 0
        outs.append((A, B, C))
    assert lib.ozk_check_split_flag(flags.data_ptr(), st) == 0
    assert lib.ozk_check_split_flag(flags.data_ptr() + 4, st) == 0
    for (_, _, C), want in zip(outs, wants):
        assert_bitwise(C.cpu().numpy(), want, "async entry")
    # data errors: NaN in B only -> flag 1; too large in A and NaN in B -> A's flag
    a = cpu.gen_eq1(2, 40, 200, 5)
    b = cpu.gen_eq1(2, 200, 30, 6)
    b[3, 4, 0] = np.nan
    A, B = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
    C = torch.empty((40, 30, 2), dtype=torch.float64, device="cuda")
    assert lib.ozk_ozaki_gemm_device_async(2, 40, 200, 30, A.data_ptr(), B.data_ptr(), 4, 0.0,
                                           C.data_ptr(), flags.data_ptr(), st) == 0
    assert lib.ozk_check_split_flag(flags.data_ptr(), st) == 0
    assert lib.ozk_check_split_flag(flags.data_ptr() + 4, st) == 2  # OZK_EPARAM
    assert b"non-finite" in lib.ozk_last_error()
    a[0, 0, :] = [2.0 ** 1000, 0.0]
    A = torch.from_numpy(a).cuda()
    assert lib.ozk_ozaki_gemm_device_async(2, 40, 200, 30, A.data_ptr(), B.data_ptr(), 4, 0.0,
                                           C.data_ptr(), flags.data_ptr(), st) == 0
    assert lib.ozk_check_split_flag(flags.data_ptr(), st) == 2
    assert b"too large" in lib.ozk_last_error()
    # argument errors come back at once
    assert lib.ozk_ozaki_gemm_device_async(2, 0, 200, 30, A.data_ptr(), B.data_ptr(), 4, 0.0,
                                           C.data_ptr(), flags.data_ptr(), st) == 1
    assert lib.ozk_ozaki_gemm_device_async(2, 40, 200, 30, A.data_ptr(), B.data_ptr(), 4, 0.0,
                                           C.data_ptr(), None, st) == 2


def test_host_api_pageable_misaligned(ozk, cpu):
    """Pageable caller buffers that are only 8-byte aligned (a DenseMatrix
    inside a larger allocation): the staging copies' streaming 16-byte stores
    handle the unaligned head and tail of every chunk; C bit-identical to the
    aligned call and to the reference rows."""
    K, m, l, n, d = 3, 2304, 300, 4104, 5
    a = cpu.gen_eq1(K, m, l, 61)
    b = cpu.gen_eq1(K, l, n, 62)

    def shifted(x):  # the same values at an address = 8 mod 16
        buf = np.empty(x.size + 1)
        v = buf[1:].reshape(x.shape)
        v[...] = x
        assert v.ctypes.data % 16 == 8
        return v

    ref = np.empty((m, n, K))
    assert ozk.lib.ozk_ozaki_gemm(K, m, l, n, a.ctypes.data, b.ctypes.data, d, 0.0,
                                  ref.ctypes.data, None) == 0, ozk.lib.ozk_last_error()
    sa, sb = shifted(a), shifted(b)
    sc = shifted(np.zeros((m, n, K)))
    assert ozk.lib.ozk_ozaki_gemm(K, m, l, n, sa.ctypes.data, sb.ctypes.data, d, 0.0,
                                  sc.ctypes.data, None) == 0, ozk.lib.ozk_last_error()
    assert_bitwise(sc, ref, "8-byte aligned pageable buffers")
    rows = np.arange(0, m, 173)
    assert_bitwise(ref[rows], cpu.ozaki_gemm(K, np.ascontiguousarray(a[rows]), b, d),
                   "sampled rows vs the reference")


def test_host_api_pageable_concurrent_and_per_device(ozk, cpu):
    """Concurrent ozk_ozaki_gemm calls from pageable buffers each take their
    own pinned slot set (the cache hands one set per call) and give the
    single-call bits; with a second GPU, a call made while device 1 is current
    stages through a slot set of device 1 (the slot events belong to one
    device) -- skipped on one GPU."""
    import ctypes
    import threading

    import torch
    K, m, l, n, d = 2, 2048, 200, 4096, 5
    a = cpu.gen_eq1(K, m, l, 51)
    b = cpu.gen_eq1(K, l, n, 52)
    ref = np.empty((m, n, K))
    assert ozk.lib.ozk_ozaki_gemm(K, m, l, n, a.ctypes.data, b.ctypes.data, d, 0.0,
                                  ref.ctypes.data, None) == 0, ozk.lib.ozk_last_error()
    outs = [np.empty((m, n, K)) for _ in range(3)]
    status = [None] * 3

    def call(i):
        status[i] = ozk.lib.ozk_ozaki_gemm(K, m, l, n, a.ctypes.data, b.ctypes.data, d, 0.0,
                                           outs[i].ctypes.data, None)

    ths = [threading.Thread(target=call, args=(i,)) for i in range(3)]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    for i in range(3):
        assert status[i] == 0
        assert_bitwise(outs[i], ref, f"concurrent pageable call {i}")
    rows = np.arange(0, m, 131)
    assert_bitwise(ref[rows], cpu.ozaki_gemm(K, np.ascontiguousarray(a[rows]), b, d),
                   "sampled rows vs the reference")
    if torch.cuda.device_count() < 2:
        return
    for dev in (1, 0, 1):  # alternate devices: a cached set must not cross devices
        c = np.empty((m, n, K))
        with torch.cuda.device(dev):
            torch.cuda.synchronize()
            st = ozk.lib.ozk_ozaki_gemm(K, m, l, n, a.ctypes.data, b.ctypes.data, d, 0.0,
                                        c.ctypes.data, None)
        assert st == 0, ozk.lib.ozk_last_error()
        assert_bitwise(c, ref, f"pageable call on device {dev}")


@pytest.mark.parametrize("K,l,devs", [(2, 100, [0, 0]), (3, 64, [0, 0, 0]), (2, 300, [0, 0])])
def test_ozaki_gemm_multi_pruning_uses_global_maxima(ozk, cpu, K, l, devs):
    """With drop_threshold > 0 every device prunes with the maxima of ALL rows
    (ozaki.hpp:194-208), including the per-device fallback path (l <= 128 or
    DMMA): device 0's rows are scaled down so its local maxima would keep a
    different pair list."""
    m, n, d = 96, 40, 8
    a = cpu.gen_eq1(K, m, l, 400 + K)
    b = cpu.gen_eq1(K, l, n, 401 + K)
    a[: m // len(devs)] *= 2.0 ** -30
    for drop in (2.0 ** -60, 2.0 ** -100):
        want = cpu.ozaki_gemm(K, a, b, d, drop)
        got, prof = ozk.ozaki_gemm_multi(a, b, d, devices=devs, drop_threshold=drop)
        assert_bitwise(got, want, f"multi pruning K={K} l={l} drop={drop}")


def test_error_precedence_matches_reference(ozk, cpu):
    """Non-finite entries outrank entries too large to shift (the reference
    scans for finiteness before any shift, ozaki.hpp:77-78 before :109), and
    A's errors come before B's (split_matrix(a) runs first)."""
    a = cpu.gen_eq1(2, 300, 300, 5)
    b = cpu.gen_eq1(2, 300, 300, 6)
    bad_nan = a.copy()
    bad_nan[7, 3, 0] = np.nan
    bad_nan[200, 9, :] = [2.0 ** 1010, 0.0]   # too large, in a later row
    with pytest.raises(ozk.param_error, match="non-finite"):
        ozk.ozaki_gemm(bad_nan, b, 4)
    huge = a.copy()
    huge[4, 4, :] = [2.0 ** 1010, 0.0]
    nan_b = b.copy()
    nan_b[1, 1, 0] = np.inf
    with pytest.raises(ozk.param_error, match="too large"):
        ozk.ozaki_gemm(huge, nan_b, 4)
    with pytest.raises(ozk.param_error, match="non-finite"):
        ozk.ozaki_gemm(a, nan_b, 4)


@pytest.mark.parametrize("K,m,l,n,d", [(2, 300, 600, 390, 6), (3, 129, 1030, 256, 9),
                                       (4, 97, 700, 130, 12), (3, 70, 96, 80, 6),
                                       (2, 2049, 600, 4200, 4)])
def test_poisoned_scratch_bitexact(ozk, cpu, monkeypatch, K, m, l, n, d):
    """Every scratch allocation filled with 0xFF (NaN words, -1 digits and
    exponents, OZK_POISON_SCRATCH=1) and the outputs pre-filled with NaN: a
    kernel reading scratch or padding it never wrote, or leaving part of C
    unwritten, changes the result.  Device and host (banded, staged) paths,
    both engines.  (compute-sanitizer is closed on this GPU pool; this is the
    stand-in for its initcheck.)"""
    import torch
    monkeypatch.setenv("OZK_POISON_SCRATCH", "1")
    a = cpu.gen_eq1(K, m, l, 800 + m)
    b = cpu.gen_eq1(K, l, n, 801 + m)
    want = cpu.ozaki_gemm(K, a, b, d)
    sh = torch.cuda.current_stream().cuda_stream
    for engine in ("auto", "dmma"):
        ozk.set_engine(engine)
        try:
            A, B = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
            C = torch.full((m, n, K), float("nan"), dtype=torch.float64, device="cuda")
            assert ozk.lib.ozk_ozaki_gemm_device(K, m, l, n, A.data_ptr(), B.data_ptr(), d, 0.0,
                                                 C.data_ptr(), sh, None) == 0
            assert_bitwise(C.cpu().numpy(), want, f"device path, poisoned, {engine}")
            c = np.full((m, n, K), np.nan)
            assert ozk.lib.ozk_ozaki_gemm(K, m, l, n, a.ctypes.data, b.ctypes.data, d, 0.0,
                                          c.ctypes.data, None) == 0
            assert_bitwise(c, want, f"host path, poisoned, {engine}")
        finally:
            ozk.set_engine("auto")
    s = ozk.split_matrix(a, d, ozk.SplitSide.cols)
    want_p, want_r = cpu.split(K, a, d, 1)
    assert_bitwise(np.stack(s.pieces), want_p, "split pieces, poisoned")
    assert_bitwise(s.residual, want_r, "split residual, poisoned")
