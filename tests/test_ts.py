"""Triple-single (TS): 3 x binary32 words per element, S = 24.

TS is NOT in the reference -- its parity is "unpinned by the
reference".  It is defined by oracle/ozk_oracle.c, which restates
the reference's generic K >= 3 algorithms with binary32 words.  This file pins
that restatement with exact arithmetic (split reconstruction, grid invariants,
exact slice products, accuracy at saturation) and checks the GPU path against
it bit for bit (tier T1) and against the exact product (tier T2 bound).
"""
import ctypes
import os
from fractions import Fraction

import numpy as np
import pytest

import oracle.exact as ex

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KW_SO = os.path.join(ROOT, "tests", "_build", "libkword_host.so")
U_TS = 2.0 ** -72  # unit roundoff of 3 x 24-bit words


def fbits(x):
    return np.ascontiguousarray(x).view(np.uint32)


def _exact(v):
    return Fraction(float(v))


# ---------------- CPU: pin the TS restatement ----------------

def test_ts_split_reconstruction_and_grid(port):
    """sum(pieces) + residual == input exactly; piece a is an integer multiple of
    2^(e_a + sigma - 24 - 1) with |piece| <= 2^e_a, e_a = ceil(log2(max |lead|))
    of the working matrix before pass a (test_ozaki.cpp:61-92, S = 24)."""
    m = port.gen_eq1_ts(9, 13, 5)
    d = 5
    for side in (0, 1):
        pieces, resid = port.split_ts(m, d, side)
        for i in range(m.shape[0]):
            for j in range(m.shape[1]):
                want = sum(_exact(w) for w in m[i, j])
                got = sum(_exact(p[i, j]) for p in pieces) + sum(_exact(w) for w in resid[i, j])
                assert got == want
        inner = m.shape[1] if side == 0 else m.shape[0]
        sigma = port.split_shift_bits(inner, 24)
        exact = [[sum(_exact(w) for w in m[i, j]) for j in range(m.shape[1])]
                 for i in range(m.shape[0])]
        for a in range(d):
            # leading word of the working matrix before pass a: the binary32
            # nearest its exact value (renormalised form)
            lead = np.array([[abs(float(np.float32(float(
                exact[i][j] - sum(_exact(pieces[b][i, j]) for b in range(a))))))
                for j in range(m.shape[1])] for i in range(m.shape[0])])
            mu = lead.max(axis=1) if side == 0 else lead.max(axis=0)
            p = pieces[a].astype(np.float64)
            for o, mo in enumerate(mu):
                vals = p[o] if side == 0 else p[:, o]
                if mo == 0:
                    assert np.all(vals == 0)
                    continue
                e = port.exponent_ceil_log2(float(mo))
                q = np.ldexp(vals, -(e + sigma - 25))
                assert np.all(q == np.trunc(q))
                assert np.all(np.abs(vals) <= np.ldexp(1.0, e))


@pytest.mark.parametrize("n,d", [(8, 4), (24, 6), (40, 10)])
def test_ts_slice_products_exact(port, n, d):
    a = port.gen_eq1_ts(n, n + 1, 10 + n)
    b = port.gen_eq1_ts(n + 1, n, 11 + n)
    pa, _ = port.split_ts(a, d, 0)
    pb, _ = port.split_ts(b, d, 1)
    for x in range(d):
        for y in range(d - x):
            _, bad = port.exact_sgemm(pa[x], pb[y])
            assert bad == 0


def test_ts_accuracy_saturates(port):
    """Accuracy improves with D and saturates near the TS unit roundoff."""
    a = port.gen_eq1_ts(24, 64, 3)
    b = port.gen_eq1_ts(64, 20, 4)
    ref = ex.exact_gemm(a.astype(np.float64), b.astype(np.float64))
    errs = []
    for d in (2, 4, 6, 8, 10, 12, 14):
        c, _, inexact = port.ozaki_gemm_ts(a, b, d, want_inexact=True)
        assert inexact == 0
        errs.append(ex.componentwise_ulp_error(c.astype(np.float64), a.astype(np.float64),
                                               b.astype(np.float64), ref, -72))
    for e0, e1 in zip(errs, errs[1:]):
        assert e1 <= e0 * 1.15 or e1 < 4.0
    assert errs[-1] <= 4.0  # |C - C_exact| <= 4 u_TS (|A||B|)_ij at saturation


def test_ts_kword_host_matches_oracle(port):
    """kw_add<3, float> (csrc/kword.cuh, host build) vs the TS restatement."""
    if not os.path.exists(KW_SO):
        import __graft_entry__
        __graft_entry__._build_test_helpers()
    lib = ctypes.CDLL(KW_SO)
    lib.kw_host_add_ts.argtypes = [ctypes.c_size_t, ctypes.c_void_p, ctypes.c_void_p,
                                   ctypes.c_void_p]
    rng = np.random.default_rng(7)
    x = port.gen_eq1_ts(100, 100, 9).reshape(-1, 3).copy()
    n = x.shape[0]
    y = (rng.standard_normal(n) * np.exp2(rng.integers(-60, 20, n))).astype(np.float32)
    sel = rng.integers(0, 8, n)
    y[sel == 0] = 0
    y[sel == 1] = -x[sel == 1, 0]
    x[sel == 2, 1:] = 0
    x[sel == 3] = 0
    y[sel == 4] = x[sel == 4, 2]
    got = np.empty_like(x)
    lib.kw_host_add_ts(n, x.ctypes.data, y.ctypes.data, got.ctypes.data)
    want = port.ts_add_float(x, y)
    assert np.array_equal(fbits(got), fbits(want))


# ---------------- GPU: bit-exact vs the TS restatement ----------------

@pytest.mark.gpu
@pytest.mark.parametrize("rows,cols,d,side", [(16, 16, 4, 0), (16, 16, 4, 1), (33, 17, 9, 0),
                                              (17, 33, 9, 1), (130, 257, 14, 1), (1, 5, 3, 0)])
def test_ts_split_bitexact(ozk, port, rows, cols, d, side):
    m = port.gen_eq1_ts(rows, cols, rows + cols)
    want_p, want_r = port.split_ts(m, d, side)
    s = ozk.split_matrix(m, d, ozk.SplitSide(side))
    assert np.array_equal(fbits(np.stack(s.pieces)), fbits(want_p))
    assert np.array_equal(fbits(s.residual), fbits(want_r))


@pytest.mark.gpu
@pytest.mark.parametrize("m,l,n,d", [(1, 1, 1, 2), (5, 7, 4, 3), (40, 40, 40, 10),
                                     (129, 200, 131, 12), (256, 256, 256, 14), (64, 300, 70, 16)])
def test_ts_ozaki_gemm_bitexact(ozk, port, m, l, n, d):
    a = port.gen_eq1_ts(m, l, 20 + m)
    b = port.gen_eq1_ts(l, n, 21 + m)
    want, np_, inexact = port.ozaki_gemm_ts(a, b, d, want_inexact=True)
    assert inexact == 0
    got, prof = ozk.ozaki_gemm(a, b, d)
    assert got.dtype == np.float32
    assert np.array_equal(fbits(got), fbits(want))
    assert prof.pairs == np_


@pytest.mark.gpu
def test_ts_accuracy_bound_gpu(ozk, port):
    a = port.gen_eq1_ts(32, 128, 5)
    b = port.gen_eq1_ts(128, 24, 6)
    ref = ex.exact_gemm(a.astype(np.float64), b.astype(np.float64))
    got, _ = ozk.ozaki_gemm(a, b, 14)
    err = ex.componentwise_ulp_error(got.astype(np.float64), a.astype(np.float64),
                                     b.astype(np.float64), ref, -72)
    assert err <= 4.0


@pytest.mark.gpu
@pytest.mark.parametrize("m,l,n", [(1, 1, 1), (5, 7, 4), (64, 64, 64), (65, 33, 130),
                                   (200, 300, 100)])
def test_ts_direct_gemm_bitexact(ozk, port, m, l, n):
    """K5 direct TS GEMM replays ozk_oracle_ts_fma bit for bit."""
    a = port.gen_eq1_ts(m, l, 30 + m)
    b = port.gen_eq1_ts(l, n, 31 + m)
    want = port.ts_direct_gemm(a, b)
    got = ozk.ts_direct_gemm(a, b)
    assert np.array_equal(fbits(got), fbits(want))


@pytest.mark.gpu
def test_ts_direct_accuracy(ozk, port):
    a = port.gen_eq1_ts(32, 128, 5)
    b = port.gen_eq1_ts(128, 24, 6)
    ref = ex.exact_gemm(a.astype(np.float64), b.astype(np.float64))
    got = ozk.ts_direct_gemm(a, b)
    err = ex.componentwise_ulp_error(got.astype(np.float64), a.astype(np.float64),
                                     b.astype(np.float64), ref, -72)
    assert err <= 16.0  # grows ~linearly with l; 2.4 at l = 64 on the CPU restatement


@pytest.mark.gpu
@pytest.mark.parametrize("eng", ["int8", "dmma"])
@pytest.mark.parametrize("m,l,n,d", [(64, 300, 70, 12), (130, 4097, 129, 15), (200, 5000, 64, 16),
                                     (33, 700, 40, 8), (40, 1025, 50, 14), (31, 1024, 33, 13)])
def test_ts_engines_bitexact(ozk, port, eng, m, l, n, d):
    """TS on both slice-product engines: INT8 uses 2 digits (l <= 1024) or a
    single digit (l > 1024: |M| <= 2^(24-sigma) <= 64)."""
    a = port.gen_eq1_ts(m, l, 40 + m)
    b = port.gen_eq1_ts(l, n, 41 + m)
    want, _, inexact = port.ozaki_gemm_ts(a, b, d, want_inexact=True)
    assert inexact == 0
    ozk.set_engine(eng)
    try:
        got, prof = ozk.ozaki_gemm(a, b, d)
    finally:
        ozk.set_engine("auto")
    assert prof.engine == eng
    assert np.array_equal(fbits(got), fbits(want))
