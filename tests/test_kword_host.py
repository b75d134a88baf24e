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


def _split_chain_cases(K, cpu, rng, rows):
    """(w, -x) pairs exactly as the split produces them: w a renormalised
    residual, x = fl(fl(w0 + tau) - tau) with tau = 2^(e + sigma), e at or above
    the binade of w0 (the row maximum may be larger), for realistic sigma (the
    split's 24..34 at l = 2..16384 and TS's 13..19) and extreme ones (1, 2),
    followed through several passes so later residuals (tails, zeros, exact
    cancellations) are covered too."""
    ws, ys = [], []
    w = cpu.gen_eq1(K, rows, 8, int(rng.integers(1, 1 << 30))).reshape(-1, K).copy()
    w[rng.random(w.shape[0]) < 0.05, 1:] = 0.0
    w *= np.exp2(rng.integers(-40, 40, w.shape[0]).astype(float))[:, None]
    # non-canonical inputs (MultiFloat::from_components_unchecked, multifloat.hpp:
    # 147-151), which the split reads in its first pass: overlapping, unordered
    # and signed-zero words
    q = w.shape[0] // 8
    w[:q, 1:] = rng.standard_normal((q, K - 1)) * np.exp2(rng.integers(-60, 4, (q, K - 1)))
    w[q:2 * q:3, 1] = -0.0
    w[q + 1:2 * q:5, K - 1] = -0.0
    w[q + 2:2 * q:7, 1:] = 0.0
    # ties: w[1] exactly half an ulp of w[0]
    t = slice(2 * q, 2 * q + q // 4)
    w[t, 1] = np.spacing(np.abs(w[t, 0])) * 0.5 * rng.choice([-1.0, 1.0], w[t, 0].shape)
    for _ in range(6):
        w0 = w[:, 0]
        nz = w0 != 0.0
        e = np.zeros(w.shape[0], dtype=np.int64)
        m, ex = np.frexp(np.abs(w0[nz]))
        e[nz] = ex - (m == 0.5)  # ceil(log2 |w0|)
        e += rng.integers(0, 4, w.shape[0])  # the row max may be larger
        sigma = rng.choice([1, 2, 13, 19, 24, 31, 33, 34, 40], w.shape[0])
        tau = np.ldexp(1.0, (e + sigma).astype(np.int64))
        x = (w0 + tau) - tau
        use = nz & (x != 0.0)
        ws.append(w[use].copy())
        ys.append(-x[use])
        w = cpu.mf_add_double(K, w, np.where(use, -x, 0.0))
    return np.concatenate(ws), np.concatenate(ys)


@pytest.mark.parametrize("K", [2, 3, 4])
def test_split_residual_update_matches_reference(ref, port, K):
    """The split's w -= x (kw_sub_piece<K, false>: K = 2 with the exact first
    two_sum, K >= 3 with the one-comparison merge and its generic fallback, see
    kword.cuh) equals the reference's MultiFloat -= double on every (w, x) pair
    the split can produce, non-canonical first-pass inputs included."""
    import __graft_entry__
    if not os.path.exists(SO):
        __graft_entry__._build_test_helpers()
    lib = ctypes.CDLL(SO)
    lib.kw_host_split_sub.argtypes = [ctypes.c_int, ctypes.c_size_t, ctypes.c_void_p,
                                      ctypes.c_void_p, ctypes.c_void_p]
    cpu = _checker(ref, port)
    rng = np.random.default_rng(2468 + K)
    x, y = _split_chain_cases(K, cpu, rng, 12_000)
    assert x.shape[0] > 200_000
    got = np.empty_like(x)
    assert lib.kw_host_split_sub(K, x.shape[0], x.ctypes.data, y.ctypes.data,
                                 got.ctypes.data) == 0
    want = cpu.mf_add_double(K, x, y)
    bad = np.flatnonzero((got.view(np.uint64) != want.view(np.uint64)).any(axis=1))
    assert bad.size == 0, (bad.size, x[bad[0]], y[bad[0]], got[bad[0]], want[bad[0]])


def test_split_residual_update_ts(port):
    """The same for TS (binary32 words, S = 24) against the C restatement."""
    import __graft_entry__
    if not os.path.exists(SO):
        __graft_entry__._build_test_helpers()
    lib = ctypes.CDLL(SO)
    lib.kw_host_split_sub_ts.argtypes = [ctypes.c_size_t, ctypes.c_void_p, ctypes.c_void_p,
                                         ctypes.c_void_p]
    rng = np.random.default_rng(1357)
    w = port.gen_eq1_ts(4000, 8, 3).reshape(-1, 3).copy()
    w *= np.exp2(rng.integers(-30, 30, w.shape[0]).astype(np.float32))[:, None]
    xs, ys = [], []
    for _ in range(5):
        w0 = w[:, 0].astype(np.float32)
        nz = w0 != 0
        e = np.zeros(w.shape[0], dtype=np.int64)
        m, ex = np.frexp(np.abs(w0[nz]))
        e[nz] = ex - (m == 0.5)
        e += rng.integers(0, 3, w.shape[0])
        sigma = rng.choice([1, 5, 13, 19], w.shape[0])
        tau = np.ldexp(np.float32(1.0), (e + sigma).astype(np.int64)).astype(np.float32)
        x = ((w0 + tau).astype(np.float32) - tau).astype(np.float32)
        use = nz & (x != 0)
        xs.append(w[use].copy())
        ys.append(-x[use])
        w = port.ts_add_float(w, np.where(use, -x, np.float32(0)).astype(np.float32))
    x = np.ascontiguousarray(np.concatenate(xs), dtype=np.float32)
    y = np.ascontiguousarray(np.concatenate(ys), dtype=np.float32)
    got = np.empty_like(x)
    lib.kw_host_split_sub_ts(x.shape[0], x.ctypes.data, y.ctypes.data, got.ctypes.data)
    want = port.ts_add_float(x, y)
    bad = np.flatnonzero((got.view(np.uint32) != want.view(np.uint32)).any(axis=1))
    assert bad.size == 0, (bad.size, x[bad[0]], y[bad[0]], got[bad[0]], want[bad[0]])


def _accum_lib():
    import __graft_entry__
    if not os.path.exists(SO):
        __graft_entry__._build_test_helpers()
    lib = ctypes.CDLL(SO)
    lib.kw_host_add_accum.argtypes = [ctypes.c_int, ctypes.c_size_t, ctypes.c_void_p,
                                      ctypes.c_void_p, ctypes.c_void_p]
    lib.kw_host_add_accum_ts.argtypes = [ctypes.c_size_t, ctypes.c_void_p, ctypes.c_void_p,
                                         ctypes.c_void_p]
    return lib


def _tail_addends(rng, x, K):
    """Addends for the last-word shortcut's bounds (kword.cuh kw_add_tail):
    around ulp(x[K-1]) / 4 (h == x[K-1]), around ulp(x[K-2]) / 2 and |x[K-2]|
    (where fl(x[K-2] + h) == x[K-2] stops holding and the merge order flips),
    -x[K-1] (h == 0) and -x[K-1] plus a little, with both signs; some x[K-1]
    become exact powers of two or zero."""
    n = x.shape[0]
    e1 = np.frexp(np.abs(x[:, K - 1]))[1] - 1
    e2 = np.frexp(np.abs(x[:, K - 2]))[1] - 1
    kind = rng.integers(0, 6, n)
    f = rng.choice([0.5, 0.999, 1.0, 1.0000001, 1.5, 2.0, 2.0 ** -30, 3.0], n)
    sgn = np.where(rng.random(n) < 0.5, -1.0, 1.0)
    y = np.ldexp(1.0, e1 - 54) * f * sgn                       # ~ ulp(x[K-1]) / 4
    y = np.where(kind == 1, np.ldexp(1.0, e2 - 53) * f * sgn, y)  # ~ ulp(x[K-2]) / 2
    y = np.where(kind == 2, x[:, K - 2] * f * -sgn, y)           # ~ |x[K-2]|
    y = np.where(kind == 3, -x[:, K - 1], y)                    # h == 0
    y = np.where(kind == 4, -x[:, K - 1] * (1 + 2.0 ** -40) + np.ldexp(1.0, e1 - 80), y)
    y = np.where(kind == 5, np.ldexp(1.0, (e1 + e2) // 2 - 53) * f * sgn, y)  # in between
    pw = rng.random(n) < 0.15
    x[pw, K - 1] = np.copysign(np.ldexp(1.0, e1[pw]), x[pw, K - 1])
    z = rng.random(n) < 0.05
    x[z, K - 1] = 0.0
    return y


@pytest.mark.parametrize("K", [2, 3, 4])
def test_accumulation_tail_shortcut_matches_reference(ref, port, K):
    """kw_add's accumulation flavour (kAccum: the last-word shortcut of
    kword.cuh kw_add_tail, taken when its conditions are checked true) equals
    the reference on reference-produced fixpoints with addends straddling every
    bound of the shortcut, on power-of-two and zero last words, on non-fixpoint
    x (the checks must refuse), and along long Ozaki-shaped chains."""
    cpu = _checker(ref, port)
    lib = _accum_lib()
    rng = np.random.default_rng(97531 + K)

    def run(x, y):
        x = np.ascontiguousarray(x)
        y = np.ascontiguousarray(y)
        got = np.empty_like(x)
        assert lib.kw_host_add_accum(K, x.shape[0], x.ctypes.data, y.ctypes.data,
                                     got.ctypes.data) == 0
        want = cpu.mf_add_double(K, x, y)
        bad = np.flatnonzero((got.view(np.uint64) != want.view(np.uint64)).any(axis=1))
        assert bad.size == 0, (bad.size, x[bad[0]], y[bad[0]], got[bad[0]], want[bad[0]])

    # reference outputs (fixpoints) with addends around every bound
    x = cpu.gen_eq1(K, 500, 100, 77).reshape(-1, K).copy()
    x = cpu.mf_add_double(K, x, rng.standard_normal(x.shape[0]) * 2.0 ** -70)
    for _ in range(4):
        xx = x.copy()
        run(xx, _tail_addends(rng, xx, K))
    # non-fixpoint x: adjacent words overlapping, sign patterns, zeros
    xn = x.copy()
    sel = rng.integers(0, 5, xn.shape[0])
    xn[sel == 0, K - 1] = xn[sel == 0, K - 2] * 0.75
    xn[sel == 1, 1] = -xn[sel == 1, 1] * 2.0 ** 60
    xn[sel == 2, K - 2] = 0.0
    xn[sel == 3, 0] = xn[sel == 3, 1] * 0.5
    run(xn, _tail_addends(rng, xn.copy(), K))
    # chains: acc += C_p with the Ozaki magnitudes 2^-20 per level
    acc_a = np.zeros((20000, K))
    acc_b = np.zeros((20000, K))
    for p in range(6 * (4 + 3 * K)):  # levels 0 .. 3K+3: past the last word
        y = rng.standard_normal(20000) * 2.0 ** (-20 * (p // 6))
        got = np.empty_like(acc_a)
        assert lib.kw_host_add_accum(K, acc_a.shape[0], acc_a.ctypes.data, y.ctypes.data,
                                     got.ctypes.data) == 0
        acc_a = got
        acc_b = cpu.mf_add_double(K, acc_b, y)
        assert np.array_equal(acc_a.view(np.uint64), acc_b.view(np.uint64)), p


def test_accumulation_tail_shortcut_ts(port):
    lib = _accum_lib()
    rng = np.random.default_rng(8642)
    acc_a = np.zeros((8000, 3), dtype=np.float32)
    acc_b = np.zeros((8000, 3), dtype=np.float32)
    for p in range(60):
        y = (rng.standard_normal(8000) * 2.0 ** (-5 * (p // 3))).astype(np.float32)
        got = np.empty_like(acc_a)
        lib.kw_host_add_accum_ts(acc_a.shape[0], acc_a.ctypes.data, y.ctypes.data,
                                 got.ctypes.data)
        acc_a = got
        acc_b = port.ts_add_float(acc_b, y)
        assert np.array_equal(acc_a.view(np.uint32), acc_b.view(np.uint32)), p
