"""K6 bit test on CPU: the device K-word "+ double" (csrc/kword.cuh, compiled
for the host with -ffp-contract=off) against the reference's
MultiFloat<K>::operator+(MultiFloat<K>, double) (multifloat.hpp:203-213),
compiled in place (oracle/_ref) -- or the C restatement when it is absent.

This is the operation both the split (w -= x) and the fused accumulation
(acc += C_ab) replay, so it decides bit-exactness of slices and of C.
"""
import ctypes
import os

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SO = os.path.join(ROOT, "tests", "_build", "libkword_host.so")


@pytest.fixture(scope="module")
def kw():
    if not os.path.exists(SO):
        import __graft_entry__
        __graft_entry__._build_test_helpers()
    lib = ctypes.CDLL(SO)
    lib.kw_host_add.argtypes = [ctypes.c_int, ctypes.c_size_t, ctypes.c_void_p, ctypes.c_void_p,
                                ctypes.c_void_p]

    def add(K, x, y):
        x = np.ascontiguousarray(x, dtype=np.float64).reshape(-1, K)
        y = np.ascontiguousarray(y, dtype=np.float64).reshape(-1)
        out = np.empty_like(x)
        assert lib.kw_host_add(K, x.shape[0], x.ctypes.data, y.ctypes.data, out.ctypes.data) == 0
        return out
    return add


def _checker(ref, port):
    return ref if ref is not None else port


def _cases(K, cpu, rng, count):
    """Adversarial (K-word, double) pairs: renormalised values from the
    reference generator, raw random words, zeros in every position, exact
    cancellations, magnitude ties with either sign, tiny/huge addends."""
    x = cpu.gen_eq1(K, count // 8, 8, int(rng.integers(1, 1 << 30))).reshape(-1, K).copy()
    y = rng.standard_normal(count) * np.exp2(rng.integers(-160, 40, count).astype(float))
    sel = rng.integers(0, 12, count)
    for i in range(count):
        s = sel[i]
        if s == 0:
            y[i] = 0.0
        elif s == 1:
            y[i] = -x[i, 0]
        elif s == 2:
            y[i] = x[i, rng.integers(0, K)] * (1 if rng.random() < .5 else -1)
        elif s == 3:
            x[i, rng.integers(0, K):] = 0.0
        elif s == 4:
            x[i] = rng.standard_normal(K) * np.exp2(rng.integers(-60, 60, K).astype(float))
        elif s == 5:
            x[i] = 0.0
        elif s == 6:
            x[i, 1:] = 0.0
            y[i] = np.nextafter(-x[i, 0], 0.0)
        elif s == 7:
            y[i] = np.ldexp(x[i, 0], -53 * int(rng.integers(1, K + 1)))
        elif s == 8:
            x[i] *= 2.0 ** -1000  # deep subnormal tails
            y[i] *= 2.0 ** -1000
        elif s == 9:
            x[i, K - 1] = -x[i, K - 1]  # non-renormalised sign pattern
        elif s == 10:
            y[i] = -0.0
    return x, y


@pytest.mark.parametrize("K", [2, 3, 4])
def test_kword_add_matches_reference(kw, ref, port, K):
    cpu = _checker(ref, port)
    rng = np.random.default_rng(1234 + K)
    x, y = _cases(K, cpu, rng, 200_000)
    got = kw(K, x, y)
    want = cpu.mf_add_double(K, x, y)
    bad = np.flatnonzero((got.view(np.uint64) != want.view(np.uint64)).any(axis=1))
    assert bad.size == 0, (f"{bad.size} mismatches; first x={x[bad[0]]} y={y[bad[0]]} "
                           f"got={got[bad[0]]} want={want[bad[0]]}")


@pytest.mark.parametrize("K", [2, 3, 4])
def test_kword_accumulation_chain(kw, ref, port, K):
    """Long chains acc += y_p as in the accumulation loop (ozaki.hpp:239-244)."""
    cpu = _checker(ref, port)
    rng = np.random.default_rng(99 + K)
    n = 5000
    acc_a = np.zeros((n, K))
    acc_b = np.zeros((n, K))
    scale = np.exp2(rng.integers(-20, 20, n).astype(float))
    for p in range(40):
        y = rng.standard_normal(n) * scale * 2.0 ** (-20 * (p // 5))
        y[rng.random(n) < 0.05] = 0.0
        acc_a = kw(K, acc_a, y)
        acc_b = cpu.mf_add_double(K, acc_b, y)
        assert np.array_equal(acc_a.view(np.uint64), acc_b.view(np.uint64)), p


@pytest.mark.parametrize("K", [2, 3, 4])
def test_kword_nonfinite(kw, ref, port, K):
    cpu = _checker(ref, port)
    x = np.zeros((6, K))
    x[:, 0] = [1.0, np.inf, -np.inf, np.nan, 1.0, 1e308]
    y = np.array([np.inf, 1.0, np.inf, 0.0, np.nan, 1e308])
    got = kw(K, x, y)
    want = cpu.mf_add_double(K, x, y)
    # NaN payloads may differ in sign bit representation only if the op order
    # differs; compare bitwise
    assert np.array_equal(got.view(np.uint64), want.view(np.uint64))


@pytest.fixture(scope="module")
def kwkw():
    lib = ctypes.CDLL(SO)
    lib.kw_host_add_kw.argtypes = [ctypes.c_int, ctypes.c_size_t, ctypes.c_void_p,
                                   ctypes.c_void_p, ctypes.c_void_p]

    def add(K, x, y):
        x = np.ascontiguousarray(x, dtype=np.float64).reshape(-1, K)
        y = np.ascontiguousarray(y, dtype=np.float64).reshape(-1, K)
        out = np.empty_like(x)
        assert lib.kw_host_add_kw(K, x.shape[0], x.ctypes.data, y.ctypes.data,
                                  out.ctypes.data) == 0
        return out
    return add


@pytest.mark.parametrize("K", [2, 3, 4])
def test_kword_add_kword_matches_reference(kwkw, ref, K):
    """MultiFloat<K> + MultiFloat<K> (multifloat.hpp:184-199), used by the LU
    trailing update's w -= update, vs the compiled reference."""
    if ref is None:
        pytest.skip("oracle/_ref not built")
    rng = np.random.default_rng(77 + K)
    x = ref.gen_eq1(K, 200, 200, 5).reshape(-1, K).copy()
    y = ref.gen_eq1(K, 200, 200, 6).reshape(-1, K).copy()
    n = x.shape[0]
    sel = rng.integers(0, 8, n)
    y[sel == 0] = -x[sel == 0]                      # exact cancellation
    y[sel == 1] = 0.0
    y[sel == 2] *= 2.0 ** -60                        # tiny addend
    y[sel == 3, 1:] = 0.0
    x[sel == 4] = -y[sel == 4] * 2.0 ** -53          # overlapping scales
    y[sel == 5] = x[sel == 5]                        # ties in the merge
    x[sel == 6, 0] = 0.0
    got = kwkw(K, x, y)
    lib = ref.lib
    lib.ref_mf_add_mf.argtypes = [ctypes.c_int, ctypes.c_size_t, ctypes.c_void_p,
                                  ctypes.c_void_p, ctypes.c_void_p]
    want = np.empty_like(x)
    assert lib.ref_mf_add_mf(K, n, x.ctypes.data, y.ctypes.data, want.ctypes.data) == 0
    bad = np.flatnonzero((got.view(np.uint64) != want.view(np.uint64)).any(axis=1))
    assert bad.size == 0, (bad.size, x[bad[0]], y[bad[0]], got[bad[0]], want[bad[0]])


@pytest.mark.parametrize("K", [2, 3, 4])
def test_kword_add_integer_compare_variant(ref, port, K):
    """The device's fast path (bit-pattern comparisons, kw_add_impl<K, true>)
    equals the reference on every input it is used for: finite words below
    2^1000 (kword.cuh Bits<>)."""
    import __graft_entry__
    if not os.path.exists(SO):
        __graft_entry__._build_test_helpers()
    lib = ctypes.CDLL(SO)
    lib.kw_host_add_int.argtypes = [ctypes.c_int, ctypes.c_size_t, ctypes.c_void_p,
                                    ctypes.c_void_p, ctypes.c_void_p]
    cpu = _checker(ref, port)
    rng = np.random.default_rng(4321 + K)
    x, y = _cases(K, cpu, rng, 200_000)
    safe = (np.abs(x) < 2.0 ** 1000).all(axis=1) & (np.abs(y) < 2.0 ** 1000)
    safe &= np.isfinite(x).all(axis=1) & np.isfinite(y)
    x, y = np.ascontiguousarray(x[safe]), np.ascontiguousarray(y[safe])
    got = np.empty_like(x)
    assert lib.kw_host_add_int(K, x.shape[0], x.ctypes.data, y.ctypes.data, got.ctypes.data) == 0
    want = cpu.mf_add_double(K, x, y)
    bad = np.flatnonzero((got.view(np.uint64) != want.view(np.uint64)).any(axis=1))
    assert bad.size == 0, (bad.size, x[bad[0]], y[bad[0]], got[bad[0]], want[bad[0]])


@pytest.mark.parametrize("K", [2, 3, 4])
def test_kword_mul_kword_matches_reference(ref, K):
    """MultiFloat<K> * MultiFloat<K> (multifloat.hpp:218-239: two_prod with FMA,
    canonical_order, sum_ordered) -- the direct K-word GEMM's multiply -- vs the
    compiled reference, incl. zeros, signs, ties and scale extremes."""
    if ref is None:
        pytest.skip("oracle/_ref not built")
    import __graft_entry__
    if not os.path.exists(SO):
        __graft_entry__._build_test_helpers()
    lib = ctypes.CDLL(SO)
    lib.kw_host_mul_kw.argtypes = [ctypes.c_int, ctypes.c_size_t, ctypes.c_void_p,
                                   ctypes.c_void_p, ctypes.c_void_p]
    rng = np.random.default_rng(500 + K)
    x = ref.gen_eq1(K, 300, 300, 9).reshape(-1, K).copy()
    y = ref.gen_eq1(K, 300, 300, 10).reshape(-1, K).copy()
    n = x.shape[0]
    sel = rng.integers(0, 10, n)
    x[sel == 0] = 0.0
    y[sel == 1, 1:] = 0.0
    y[sel == 2] = -x[sel == 2]
    x[sel == 3] *= 2.0 ** -900
    y[sel == 4] *= 2.0 ** 700
    x[sel == 5] = -x[sel == 5]
    x[sel == 6, K - 1] = 0.0
    y[sel == 7] = x[sel == 7]
    got = np.empty_like(x)
    assert lib.kw_host_mul_kw(K, n, x.ctypes.data, y.ctypes.data, got.ctypes.data) == 0
    rl = ref.lib
    rl.ref_mf_mul_mf.argtypes = [ctypes.c_int, ctypes.c_size_t, ctypes.c_void_p,
                                 ctypes.c_void_p, ctypes.c_void_p]
    want = np.empty_like(x)
    assert rl.ref_mf_mul_mf(K, n, x.ctypes.data, y.ctypes.data, want.ctypes.data) == 0
    bad = np.flatnonzero((got.view(np.uint64) != want.view(np.uint64)).any(axis=1))
    assert bad.size == 0, (bad.size, x[bad[0]], y[bad[0]], got[bad[0]], want[bad[0]])


@pytest.mark.parametrize("K", [3, 4])
def test_kword_add_fp_compare_flavour(ref, port, K):
    """kw_add<K, double, false> -- the fast path with FP64 comparisons, as the
    split uses it -- equals the reference on the adversarial set."""
    import __graft_entry__
    if not os.path.exists(SO):
        __graft_entry__._build_test_helpers()
    lib = ctypes.CDLL(SO)
    lib.kw_host_add_fpcmp.argtypes = [ctypes.c_int, ctypes.c_size_t, ctypes.c_void_p,
                                      ctypes.c_void_p, ctypes.c_void_p]
    cpu = _checker(ref, port)
    rng = np.random.default_rng(8765 + K)
    x, y = _cases(K, cpu, rng, 200_000)
    got = np.empty_like(x)
    assert lib.kw_host_add_fpcmp(K, x.shape[0], x.ctypes.data, y.ctypes.data, got.ctypes.data) == 0
    want = cpu.mf_add_double(K, x, y)
    bad = np.flatnonzero((got.view(np.uint64) != want.view(np.uint64)).any(axis=1))
    assert bad.size == 0, (bad.size, x[bad[0]], y[bad[0]], got[bad[0]], want[bad[0]])
