"""Exact (big-integer) oracle -- TEST INFRASTRUCTURE ONLY.

Restates the reference's GMP oracle with Python integers (GMP headers are not
available here):

* ``BigFloat`` (``proj/include/mpmat/oracle.hpp:18-54``, ``proj/src/oracle.cpp``):
  an exact dyadic ``mant * 2**exp``; here a ``(mant, exp)`` pair of Python ints.
* ``exact_gemm`` (``oracle.hpp:59-74``) and ``exact_gemm_f64``
  (``oracle.cpp:96-110``): exact products.
* ``to_double`` (``oracle.cpp:62-78``): keeps the top 64 bits (truncating
  ``mpz_tdiv_q_2exp``) then ``mpz_get_d`` (truncating) -> the value truncated
  toward zero to 53 significant bits.
* ``max_rel_error`` (``oracle.hpp:81-92``): max over elements of
  ``|c - ref| / |ref|`` (``|c|`` absolutely when ``ref == 0``), each side
  converted with ``to_double`` and divided in binary64.

Pure-Python loops: for small matrices only (n <= ~64 for K-word inputs).
"""
from __future__ import annotations

import math

import numpy as np


def dyadic(x: float) -> tuple[int, int]:
    """Exact (mant, exp) of a binary64 value, oracle.cpp:8-16."""
    if x == 0.0:
        return 0, 0
    if not math.isfinite(x):
        raise ValueError("non-finite")
    m, e = math.frexp(x)
    return int(m * (1 << 53)), e - 53


def add(a: tuple[int, int], b: tuple[int, int]) -> tuple[int, int]:
    (ma, ea), (mb, eb) = a, b
    if mb == 0:
        return a
    if ma == 0:
        return b
    if ea == eb:
        r = (ma + mb, ea)
    elif ea > eb:
        r = ((ma << (ea - eb)) + mb, eb)
    else:
        r = (ma + (mb << (eb - ea)), ea)
    return (0, 0) if r[0] == 0 else r


def mul(a, b):
    if a[0] == 0 or b[0] == 0:
        return (0, 0)
    return (a[0] * b[0], a[1] + b[1])


def neg(a):
    return (-a[0], a[1])


def of_words(words) -> tuple[int, int]:
    """BigFloat(MultiFloat<K>) (oracle.hpp:27-30): exact sum of the K words."""
    r = (0, 0)
    for w in words:
        r = add(r, dyadic(float(w)))
    return r


def to_double(a) -> float:
    """BigFloat::to_double (oracle.cpp:62-78): truncation toward zero to 53 bits."""
    m, e = a
    if m == 0:
        return 0.0
    sign = -1 if m < 0 else 1
    m = abs(m)
    bits = m.bit_length()
    if bits > 53:
        m >>= bits - 53
        e += bits - 53
    total = e
    if total > 2000:
        return sign * math.inf
    if total < -2000:
        return sign * 0.0
    return sign * math.ldexp(float(m), total)


def exact_gemm(a: np.ndarray, b: np.ndarray) -> list:
    """oracle.hpp:59-74 on K-word AoS arrays a (m,l,K), b (l,n,K); row-major list."""
    m, l = a.shape[0], a.shape[1]
    n = b.shape[1]
    ea = [[of_words(a[i, k]) for k in range(l)] for i in range(m)]
    eb = [[of_words(b[k, j]) for j in range(n)] for k in range(l)]
    # common exponent per matrix -> plain integer dot products
    emin_a = min((x[1] for row in ea for x in row if x[0]), default=0)
    emin_b = min((x[1] for row in eb for x in row if x[0]), default=0)
    ia = [[(x[0] << (x[1] - emin_a)) if x[0] else 0 for x in row] for row in ea]
    ib = [[(x[0] << (x[1] - emin_b)) if x[0] else 0 for x in row] for row in eb]
    out = []
    for i in range(m):
        ai = ia[i]
        for j in range(n):
            s = 0
            for k in range(l):
                if ai[k]:
                    s += ai[k] * ib[k][j]
            out.append((s, emin_a + emin_b) if s else (0, 0))
    return out


def max_rel_error(c: np.ndarray, ref: list) -> float:
    """oracle.hpp:81-92."""
    K = c.shape[-1]
    flat = c.reshape(-1, K)
    worst = 0.0
    for i, r in enumerate(ref):
        diff = add(of_words(flat[i]), neg(r))
        ad = (abs(diff[0]), diff[1])
        if r[0] == 0:
            err = to_double(ad)
        else:
            err = to_double(ad) / to_double((abs(r[0]), r[1]))
        if err > worst:
            worst = err
    return worst


def componentwise_ulp_error(c: np.ndarray, a: np.ndarray, b: np.ndarray, ref: list,
                            ulp_exp: int) -> float:
    """max_ij |C_ij - C_exact_ij| / (2**ulp_exp * (|A||B|)_ij) -- the T2 parity bound
    of SURVEY.md §8 (u_L = 2^-106 / 2^-159 / 2^-212 for DD / TD / QD)."""
    m, l, n = a.shape[0], a.shape[1], b.shape[1]
    K = c.shape[-1]
    absa = np.abs(a[..., 0]).astype(np.float64)
    absb = np.abs(b[..., 0]).astype(np.float64)
    # |A||B| from the leading words, inflated by 2^-50 to bound the tails
    mag = (absa @ absb) * (1.0 + 2.0 ** -50)
    flat = c.reshape(-1, K)
    worst = 0.0
    for idx, r in enumerate(ref):
        diff = add(of_words(flat[idx]), neg(r))
        if diff[0] == 0:
            continue
        i, j = divmod(idx, n)
        val = abs(to_double((abs(diff[0]), diff[1])))
        den = mag[i, j]
        if den == 0.0:
            return math.inf
        worst = max(worst, math.ldexp(val / den, -ulp_exp))
    return worst
