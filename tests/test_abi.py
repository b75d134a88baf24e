"""The C-ABI library loads, exports every symbol include/ozk.h declares, and
its host-side logic (KATs, argument validation) behaves like the reference --
all without a GPU (no compute call reaches the device here)."""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    src = open(os.path.join(ROOT, "include", "ozk.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ozk_[a-z0-9_]+)\s*\(", src)))


def test_header_symbols_exported():
    from paper_2301_09960_b200._lib import LIB_PATH, SIGNATURES
    lib = ctypes.CDLL(LIB_PATH)
    names = declared_functions()
    assert len(names) >= 15
    for name in names:
        assert hasattr(lib, name), f"{name} declared in ozk.h but not exported"
    # the Python binding covers exactly the header
    assert sorted(SIGNATURES) == names


def test_header_has_no_torch_types():
    src = open(os.path.join(ROOT, "include", "ozk.h")).read()
    code = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    assert "torch" not in code.lower()
    assert not re.search(r"\bat::|\bc10::|Tensor", code)


def test_split_shift_bits_kats():
    """test_ozaki.cpp:130-138 and SURVEY Appendix B."""
    import paper_2301_09960_b200 as ozk
    kat = {1024: 32, 1: 27, 2: 27, 8: 28, 9: 29, 256: 31, 5: 28, 4096: 33, 8192: 33, 16384: 34}
    for l, s in kat.items():
        assert ozk.split_shift_bits(l) == s, l


def test_int8_digit_counts():
    """ozk_int8_digits: digits per slice integer |M| <= 2^(S+1-sigma) in signed
    base 256 (csrc/api.cu int8_digits), 0 where the engine does not apply."""
    from paper_2301_09960_b200._lib import lib
    for l, nd in [(1, 0), (128, 0), (129, 3), (512, 3), (4096, 3), (8192, 3), (16384, 3), (43689, 3),
                  (43690, 0)]:
        assert lib.ozk_int8_digits(2, l, 6) == nd, l
        assert lib.ozk_int8_digits(4, l, 12) == nd, l
    # TS (S = 24): 2 digits up to l = 1024 (|M| <= 2^(24 - sigma)), 1 beyond
    for l, nd in [(16, 2), (1024, 2), (1025, 1), (4096, 1), (8192, 1), (43690, 0)]:
        assert lib.ozk_int8_digits(0x103, l, 15) == nd, l
    assert lib.ozk_int8_digits(2, 8192, 1) == 0  # D = 1 is the leading image: DMMA path
    assert lib.ozk_int8_digits(7, 8192, 6) == 0  # not a format


def test_exponent_ceil_log2(port):
    """test_ozaki.cpp:111-128: table + 20k random samples vs a linear-scan oracle."""
    import paper_2301_09960_b200 as ozk
    for x, e in [(1.0, 0), (8.0, 3), (9.0, 4), (0.5, -1), (0.75, 0)]:
        assert ozk.exponent_ceil_log2(x) == e
    rng = np.random.default_rng(55)
    for _ in range(20000):
        x = np.ldexp(rng.random() + 1e-12, int(rng.integers(0, 600)) - 300)
        e = ozk.exponent_ceil_log2(x)
        assert np.ldexp(1.0, e) >= x and np.ldexp(1.0, e - 1) < x
        assert e == port.exponent_ceil_log2(x)


def test_argument_errors_without_gpu():
    """Error conditions and their order (ozaki.hpp:184-186, dense_matrix.hpp:23)
    are decided on the host before any device work."""
    import paper_2301_09960_b200 as ozk
    a = np.zeros((2, 2, 2))
    with pytest.raises(ozk.shape_error):
        ozk.ozaki_gemm(a, np.zeros((3, 2, 2)), 2)
    with pytest.raises(ozk.param_error):
        ozk.ozaki_gemm(a, a, 0)
    with pytest.raises(ozk.param_error):
        ozk.ozaki_gemm(a, a, 2, drop_threshold=-1.0)
    with pytest.raises(ozk.param_error):
        ozk.ozaki_gemm(np.zeros((2, 2, 5)), np.zeros((2, 2, 5)), 2)
    lib = ozk.lib
    assert lib.ozk_ozaki_gemm(2, 0, 2, 2, None, None, 2, 0.0, None, None) == 1  # zero dim first
    assert lib.ozk_ozaki_gemm(2, 2, 2, 2, None, None, 0, 0.0, None, None) == 2
    assert lib.ozk_ozaki_gemm(2, 2, 2, 2, None, None, 2, -1.0, None, None) == 2
    assert lib.ozk_ozaki_gemm(7, 2, 2, 2, None, None, 2, 0.0, None, None) == 2
    assert lib.ozk_split(2, 2, 2, None, 0, 0, None, None) == 2
    assert b"split count" in lib.ozk_last_error()
    # the one-process multi-GPU entry point checks the same arguments first
    assert lib.ozk_ozaki_gemm_multi(2, 2, None, 0, 2, 2, None, None, 2, 0.0, None, None) == 1
    assert lib.ozk_ozaki_gemm_multi(2, 2, None, 2, 2, 2, None, None, 0, 0.0, None, None) == 2
    assert lib.ozk_ozaki_gemm_multi(2, 0, None, 2, 2, 2, None, None, 2, 0.0, None, None) == 2
    assert b"devices" in lib.ozk_last_error()
    with pytest.raises(ozk.shape_error):
        ozk.ozaki_gemm_multi(a, np.zeros((3, 2, 2)), 2, devices=[0])
    # round-2 entry points: argument errors before any device work
    assert lib.ozk_accumulate_products(7, 2, 2, None, 0, None) == 2
    assert lib.ozk_accumulate_products(2, 0, 2, None, 0, None) == 1
    assert lib.ozk_accumulate_products(2, 2, 2, None, -1, None) == 2
    assert lib.ozk_split_digits_device_async(2, 2, 2, 2, None, 0, 0, None, 16, 2, None, None,
                                             None, None) == 2
    assert lib.ozk_split_digits_device_async(2, 300, 300, 300, None, 3, 0, None, 304, 300,
                                             None, None, None, None) == 2  # null outputs
    # null operands are refused before any device work (after the shape and
    # parameter checks, which keep the reference's order)
    assert lib.ozk_ozaki_gemm(2, 2, 2, 2, None, None, 2, 0.0, None, None) == 2
    assert b"null pointer" in lib.ozk_last_error()
    assert lib.ozk_ozaki_gemm_device(2, 2, 2, 2, None, None, 2, 0.0, None, None, None) == 2
    assert lib.ozk_split(2, 2, 2, None, 2, 0, None, None) == 2
    assert b"null pointer" in lib.ozk_last_error()
    assert lib.ozk_direct_gemm(2, 2, 2, 2, None, None, None) == 2
    assert lib.ozk_backend_gemm(2, 2, 2, None, None, None) == 2
    assert lib.ozk_lu_trailing_update(2, 2, 2, 2, None, 2, None, 2, None, 2, 2) == 2
    assert lib.ozk_ozaki_gemm_multi(2, 1, None, 2, 2, 2, None, None, 2, 0.0, None, None) == 2
    assert b"null pointer" in lib.ozk_last_error()
    # a caller's backend is honoured, with the reference's argument checks first
    with pytest.raises(ozk.param_error):
        ozk.ozaki_gemm(a, a, 0, backend=lambda x, y: x @ y)
    with pytest.raises(ozk.shape_error):
        ozk.ozaki_gemm(a, np.zeros((3, 2, 2)), 2, backend=lambda x, y: x @ y)


def test_pair_list_matches_reference_order(port):
    """ozaki.hpp:198-221: alpha-major triangular list with drop pruning."""
    import paper_2301_09960_b200 as ozk
    rng = np.random.default_rng(3)
    for d in (1, 2, 3, 6, 12, 32, 40, 70):  # D > 32: pair lists run as several launches
        amax = np.sort(rng.random(d))[::-1] * np.exp2(-20.0 * np.arange(d))
        bmax = np.sort(rng.random(d))[::-1] * np.exp2(-20.0 * np.arange(d))
        for drop in (0.0, 2.0 ** -60, 2.0 ** -30, 0.5):
            buf = (ctypes.c_int * (2 * d * d))()
            cnt = ctypes.c_int(0)
            st = ozk.lib.ozk_pair_list(d, amax.ctypes.data, bmax.ctypes.data, drop, buf,
                                       ctypes.byref(cnt))
            assert st == 0
            got = np.array(buf[: 2 * cnt.value]).reshape(-1, 2)
            want = port.pair_list(d, amax, bmax, drop)
            assert np.array_equal(got, want)
            if drop == 0.0:
                assert cnt.value == d * (d + 1) // 2


def test_product_path_has_no_cpu_fallback():
    """The product package never imports the oracle and refuses to load
    without libozk.so."""
    pkg = os.path.join(ROOT, "paper_2301_09960_b200")
    for fn in os.listdir(pkg):
        if fn.endswith(".py"):
            src = open(os.path.join(pkg, fn)).read()
            assert "import oracle" not in src and "from oracle" not in src, fn
    from paper_2301_09960_b200 import _lib
    with pytest.raises(ImportError):
        _lib.load(os.path.join(ROOT, "does-not-exist.so"))


def test_auto_split_policy():
    """Automatic D: ceil(S*K / (S - sigma)) + 2 slices and pair
    pruning at 2^-(S*K + ceil(log2 l) + 2)."""
    import paper_2301_09960_b200 as ozk
    assert ozk.auto_split_policy(2, 8192) == (8, 2.0 ** -121)
    assert ozk.auto_split_policy(3, 8192) == (10, 2.0 ** -174)
    assert ozk.auto_split_policy(4, 8192) == (13, 2.0 ** -227)
    assert ozk.auto_split_policy(0x103, 8192) == (17, 2.0 ** -87)
    assert ozk.auto_split_policy(2, 1) == (7, 2.0 ** -108)   # sigma = 27: 26 bits per slice
    assert ozk.auto_split_policy(7, 8192) == (0, 0.0)


def _plan(fmt, m, n, l, d, block_cols, gr, gc, clusters, max_bands=8):
    from paper_2301_09960_b200._lib import lib
    starts = (ctypes.c_size_t * (max_bands + 1))()
    nb = lib.ozk_plan_row_bands(fmt, m, n, l, d, block_cols, gr, gc, clusters, 2, starts,
                                max_bands)
    return nb, list(starts[: nb + 1]) if nb > 0 else []


def _waves(rows, gr, n, gc, clusters):
    r = -(-rows // gr)
    return -(-(r * -(-n // gc)) // clusters)


@pytest.mark.parametrize("fmt,gr", [(2, 128), (3, 96), (4, 96), (0x103, 224)])
def test_row_band_plan_n8192(fmt, gr):
    """ozk_ozaki_gemm's host schedule (csrc/api.cu plan_bands) at n = 8192 on the
    B200 geometry (74 two-SM clusters, 128-column tiles): the bands cover every
    row once, in whole cluster rows except the end, band 0 is a short first
    wait (<= m/6), the last band is short (its C copy is the exposed tail), and
    the total GEMM waves are within one wave of 8 equal bands' (fewer for TD)."""
    m = n = l = 8192
    d = {2: 6, 3: 9, 4: 12, 0x103: 15}[fmt]
    nb, st = _plan(fmt, m, n, l, d, 2048, gr, 128, 74)
    assert 2 <= nb <= 8, st
    assert st[0] == 0 and st[-1] == m and all(a < b for a, b in zip(st, st[1:])), st
    assert all(x % gr == 0 for x in st[1:-1]), st
    assert st[1] <= m // 6 + gr, st
    planned = sum(_waves(b - a, gr, n, 128, 74) for a, b in zip(st, st[1:]))
    equal = sum(_waves(m * (q + 1) // 8 - m * q // 8, gr, n, 128, 74) for q in range(8))
    assert planned <= equal + 1, (planned, equal, st)
    if fmt == 3:
        assert planned < equal, (planned, equal, st)
    assert st[-1] - st[-2] <= m // 16, st
    # within 3 waves of the monolithic GEMM's ceil(tiles / clusters)
    assert planned <= _waves(m, gr, n, 128, 74) + 3, (planned, st)


def test_row_band_plan_edges():
    nb, st = _plan(3, 1000, 8192, 8192, 9, 2048, 96, 128, 74)
    assert (nb, st) == (1, [0, 1000])  # m < 2048: one band
    nb, st = _plan(3, 4097, 4101, 140, 3, 1152, 96, 128, 74)
    assert nb >= 1 and st[-1] == 4097 and all(a < b for a, b in zip(st, st[1:]))
    from paper_2301_09960_b200._lib import lib
    starts = (ctypes.c_size_t * 9)()
    assert lib.ozk_plan_row_bands(3, 8192, 8192, 8192, 9, 2048, 0, 128, 74, 2, starts, 8) == -1
    assert lib.ozk_plan_row_bands(9, 8192, 8192, 8192, 9, 2048, 96, 128, 74, 2, starts, 8) == -1
    assert lib.ozk_plan_row_bands(3, 8192, 8192, 8192, 9, 2048, 96, 128, 74, 2, starts, 1) == -1
