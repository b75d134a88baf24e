"""CPU checkers for the Ozaki hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference``) may import this package, and
only as the checker or the timed CPU baseline.  The product library
(``paper_2301_09960_b200``) never imports it and has no CPU fallback.

Two checkers are exposed through ctypes:

* :data:`port` -- ``oracle/_build/libozk_oracle.so``, a plain-C restatement of
  the reference hot path (``oracle/ozk_oracle.c``, every function cites the
  reference file:line it restates).  Always buildable (gcc only).
* :data:`ref` -- ``oracle/_ref/libref_oracle.so``, the UNMODIFIED reference
  (``/root/reference/proj``) compiled in place with its own flags by
  ``oracle/Makefile``.  Built in the development container, shipped prebuilt to
  the GPU box (``/root/reference`` does not exist there); ``None`` when absent.

Both expose the same Python surface (:class:`CpuOzaki`), so parity tests can
run against either.  ``oracle.exact`` restates the GMP oracle
(``proj/include/mpmat/oracle.hpp:81-92``, ``proj/src/oracle.cpp:62-78``) with
Python integers.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "_build", "libozk_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libref_oracle.so")
REF_SRC = "/root/reference/proj"

_c_size = ctypes.c_size_t
_dp = ctypes.POINTER(ctypes.c_double)
_ip = ctypes.POINTER(ctypes.c_int)
_lp = ctypes.POINTER(ctypes.c_long)


def build(ref: bool | None = None) -> None:
    """Compile the C restatement and, when the reference tree exists, oracle/_ref."""
    subprocess.run(["make", "-s", "-C", HERE, "port"], check=True)
    if ref is None:
        ref = os.path.isdir(REF_SRC)
    if ref:
        subprocess.run(["make", "-s", "-C", HERE, "ref"], check=True)


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(_dp)


class OracleError(RuntimeError):
    def __init__(self, status: int, what: str):
        super().__init__(f"{what}: status {status}")
        self.status = status


class CpuOzaki:
    """Common numpy surface over the port or the compiled reference."""

    kind = "?"

    def gen_eq1(self, K: int, m: int, n: int, seed: int) -> np.ndarray:
        raise NotImplementedError

    def split(self, K, mat, d, side):
        raise NotImplementedError

    def ozaki_gemm(self, K, a, b, d, drop=0.0):
        raise NotImplementedError

    def mf_add_double(self, K, x, y):
        raise NotImplementedError


class Port(CpuOzaki):
    """ctypes view of oracle/_build/libozk_oracle.so (C restatement)."""

    kind = "port"

    def __init__(self, path: str = PORT_SO):
        lib = ctypes.CDLL(path)
        lib.ozk_oracle_gen_eq1.argtypes = [ctypes.c_int, _c_size, _c_size, ctypes.c_uint64, _dp]
        lib.ozk_oracle_split.argtypes = [ctypes.c_int, _c_size, _c_size, _dp, ctypes.c_int,
                                         ctypes.c_int, _dp, _dp]
        lib.ozk_oracle_ozaki_gemm.argtypes = [ctypes.c_int, _c_size, _c_size, _c_size, _dp, _dp,
                                              ctypes.c_int, ctypes.c_double, _dp, _ip, _lp]
        lib.ozk_oracle_mf_add_double.argtypes = [ctypes.c_int, _dp, ctypes.c_double, _dp]
        lib.ozk_oracle_exponent_ceil_log2.argtypes = [ctypes.c_double]
        lib.ozk_oracle_split_shift_bits.argtypes = [_c_size, ctypes.c_int]
        lib.ozk_oracle_exact_dgemm.argtypes = [_c_size, _c_size, _c_size, _dp, _dp, _dp]
        lib.ozk_oracle_exact_dgemm.restype = ctypes.c_long
        lib.ozk_oracle_dgemm.argtypes = [_c_size, _c_size, _c_size, _dp, _dp, _dp]
        lib.ozk_oracle_pair_list.argtypes = [ctypes.c_int, _dp, _dp, ctypes.c_double, _ip]
        lib.ozk_oracle_replay_elements.argtypes = [ctypes.c_int, _c_size, _c_size, _c_size, _dp,
                                                   _dp, ctypes.c_int, _ip, _c_size, _lp, _lp,
                                                   _dp, _lp]
        lib.ozk_oracle_xoshiro_u64.argtypes = [ctypes.c_uint64, _c_size,
                                               ctypes.POINTER(ctypes.c_uint64)]
        _fp = ctypes.c_void_p
        lib.ozk_oracle_gen_eq1_ts.argtypes = [_c_size, _c_size, ctypes.c_uint64, _fp]
        lib.ozk_oracle_split_ts.argtypes = [_c_size, _c_size, _fp, ctypes.c_int, ctypes.c_int,
                                            _fp, _fp]
        lib.ozk_oracle_ozaki_gemm_ts.argtypes = [_c_size, _c_size, _c_size, _fp, _fp,
                                                 ctypes.c_int, ctypes.c_double, _fp, _ip, _lp]
        lib.ozk_oracle_ts_add_float.argtypes = [_fp, ctypes.c_float, _fp]
        lib.ozk_oracle_exact_sgemm.argtypes = [_c_size, _c_size, _c_size, _fp, _fp, _fp]
        lib.ozk_oracle_exact_sgemm.restype = ctypes.c_long
        lib.ozk_oracle_ts_direct_gemm.argtypes = [_c_size, _c_size, _c_size, _fp, _fp, _fp]
        lib.ozk_oracle_gen_spread.argtypes = [ctypes.c_int, _c_size, _c_size, ctypes.c_uint64,
                                              ctypes.c_int, _dp]
        self.lib = lib

    def gen_eq1(self, K, m, n, seed):
        out = np.empty((m, n, K), dtype=np.float64)
        self.lib.ozk_oracle_gen_eq1(K, m, n, seed, _ptr(out))
        return out

    def gen_spread(self, K, m, n, seed, spread):
        """Ill-conditioned inputs (config 5): Eq. (1) values scaled by 2^U[-s, s]."""
        out = np.empty((m, n, K), dtype=np.float64)
        self.lib.ozk_oracle_gen_spread(K, m, n, seed, spread, _ptr(out))
        return out

    def xoshiro(self, seed, count):
        out = np.empty(count, dtype=np.uint64)
        self.lib.ozk_oracle_xoshiro_u64(seed, count,
                                        out.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)))
        return out

    def split(self, K, mat, d, side):
        mat = np.ascontiguousarray(mat, dtype=np.float64)
        rows, cols = mat.shape[0], mat.shape[1]
        pieces = np.zeros((max(d, 1), rows, cols), dtype=np.float64)
        resid = np.empty_like(mat)
        st = self.lib.ozk_oracle_split(K, rows, cols, _ptr(mat), d, side, _ptr(pieces),
                                       _ptr(resid))
        if st:
            raise OracleError(st, "split")
        return pieces, resid

    def ozaki_gemm(self, K, a, b, d, drop=0.0, want_inexact=False):
        a = np.ascontiguousarray(a, dtype=np.float64)
        b = np.ascontiguousarray(b, dtype=np.float64)
        m, l = a.shape[0], a.shape[1]
        if b.shape[0] != l:
            raise OracleError(1, "ozaki_gemm")
        n = b.shape[1]
        c = np.zeros((m, n, K), dtype=np.float64)
        np_ = ctypes.c_int(0)
        inex = ctypes.c_long(0)
        st = self.lib.ozk_oracle_ozaki_gemm(K, m, l, n, _ptr(a), _ptr(b), d, drop, _ptr(c),
                                            ctypes.byref(np_), ctypes.byref(inex))
        if st:
            raise OracleError(st, "ozaki_gemm")
        if want_inexact:
            return c, np_.value, inex.value
        return c

    def mf_add_double(self, K, x, y):
        x = np.ascontiguousarray(x, dtype=np.float64).reshape(-1, K)
        y = np.ascontiguousarray(y, dtype=np.float64).reshape(-1)
        out = np.empty_like(x)
        r = (ctypes.c_double * K)()
        for i in range(x.shape[0]):
            self.lib.ozk_oracle_mf_add_double(K, _ptr(x[i]), float(y[i]), r)
            out[i] = np.frombuffer(r, dtype=np.float64)
        return out

    def exact_dgemm(self, a, b):
        a = np.ascontiguousarray(a, dtype=np.float64)
        b = np.ascontiguousarray(b, dtype=np.float64)
        c = np.empty((a.shape[0], b.shape[1]), dtype=np.float64)
        bad = self.lib.ozk_oracle_exact_dgemm(a.shape[0], a.shape[1], b.shape[1], _ptr(a),
                                              _ptr(b), _ptr(c))
        return c, bad

    def pair_list(self, d, amax, bmax, drop):
        amax = np.ascontiguousarray(amax, dtype=np.float64)
        bmax = np.ascontiguousarray(bmax, dtype=np.float64)
        pairs = np.zeros(2 * d * d, dtype=np.int32)
        np_ = self.lib.ozk_oracle_pair_list(d, _ptr(amax), _ptr(bmax), drop,
                                            pairs.ctypes.data_as(_ip))
        return pairs[: 2 * np_].reshape(-1, 2)

    def replay_elements(self, K, pa, pb, pairs, ii, jj):
        """C(i,j) for sampled elements from slices (pa: d x m x l, pb: d x l x n)."""
        pa = np.ascontiguousarray(pa, dtype=np.float64)
        pb = np.ascontiguousarray(pb, dtype=np.float64)
        pairs = np.ascontiguousarray(pairs, dtype=np.int32).reshape(-1)
        ii = np.ascontiguousarray(ii, dtype=np.int64)
        jj = np.ascontiguousarray(jj, dtype=np.int64)
        out = np.zeros((len(ii), K), dtype=np.float64)
        bad = ctypes.c_long(0)
        self.lib.ozk_oracle_replay_elements(K, pa.shape[1], pa.shape[2], pb.shape[2], _ptr(pa),
                                            _ptr(pb), len(pairs) // 2,
                                            pairs.ctypes.data_as(_ip), len(ii),
                                            ii.ctypes.data_as(_lp), jj.ctypes.data_as(_lp),
                                            _ptr(out), ctypes.byref(bad))
        return out, bad.value

    def exponent_ceil_log2(self, x):
        return self.lib.ozk_oracle_exponent_ceil_log2(x)

    def split_shift_bits(self, inner, short_bits=53):
        return self.lib.ozk_oracle_split_shift_bits(inner, short_bits)

    # ---- TS (triple-single, binary32 words; defined by this restatement) ----
    def gen_eq1_ts(self, m, n, seed):
        out = np.empty((m, n, 3), dtype=np.float32)
        self.lib.ozk_oracle_gen_eq1_ts(m, n, seed, out.ctypes.data)
        return out

    def split_ts(self, mat, d, side):
        mat = np.ascontiguousarray(mat, dtype=np.float32)
        rows, cols = mat.shape[0], mat.shape[1]
        pieces = np.zeros((max(d, 1), rows, cols), dtype=np.float32)
        resid = np.empty_like(mat)
        st = self.lib.ozk_oracle_split_ts(rows, cols, mat.ctypes.data, d, side,
                                          pieces.ctypes.data, resid.ctypes.data)
        if st:
            raise OracleError(st, "split_ts")
        return pieces, resid

    def ozaki_gemm_ts(self, a, b, d, drop=0.0, want_inexact=False):
        a = np.ascontiguousarray(a, dtype=np.float32)
        b = np.ascontiguousarray(b, dtype=np.float32)
        m, l, n = a.shape[0], a.shape[1], b.shape[1]
        c = np.zeros((m, n, 3), dtype=np.float32)
        np_ = ctypes.c_int(0)
        inex = ctypes.c_long(0)
        st = self.lib.ozk_oracle_ozaki_gemm_ts(m, l, n, a.ctypes.data, b.ctypes.data, d, drop,
                                               c.ctypes.data, ctypes.byref(np_),
                                               ctypes.byref(inex))
        if st:
            raise OracleError(st, "ozaki_gemm_ts")
        if want_inexact:
            return c, np_.value, inex.value
        return c

    def ts_add_float(self, x, y):
        x = np.ascontiguousarray(x, dtype=np.float32).reshape(-1, 3)
        y = np.ascontiguousarray(y, dtype=np.float32).reshape(-1)
        out = np.empty_like(x)
        r = np.empty(3, dtype=np.float32)
        for i in range(x.shape[0]):
            xi = np.ascontiguousarray(x[i])
            self.lib.ozk_oracle_ts_add_float(xi.ctypes.data, ctypes.c_float(float(y[i])),
                                             r.ctypes.data)
            out[i] = r
        return out

    def ts_direct_gemm(self, a, b):
        a = np.ascontiguousarray(a, dtype=np.float32)
        b = np.ascontiguousarray(b, dtype=np.float32)
        c = np.empty((a.shape[0], b.shape[1], 3), dtype=np.float32)
        self.lib.ozk_oracle_ts_direct_gemm(a.shape[0], a.shape[1], b.shape[1], a.ctypes.data,
                                           b.ctypes.data, c.ctypes.data)
        return c

    def exact_sgemm(self, a, b):
        a = np.ascontiguousarray(a, dtype=np.float32)
        b = np.ascontiguousarray(b, dtype=np.float32)
        c = np.empty((a.shape[0], b.shape[1]), dtype=np.float32)
        bad = self.lib.ozk_oracle_exact_sgemm(a.shape[0], a.shape[1], b.shape[1], a.ctypes.data,
                                              b.ctypes.data, c.ctypes.data)
        return c, bad


class Ref(CpuOzaki):
    """ctypes view of oracle/_ref/libref_oracle.so (reference compiled in place)."""

    kind = "reference"

    def __init__(self, path: str = REF_SO):
        lib = ctypes.CDLL(path)
        lib.ref_set_threads.argtypes = [ctypes.c_int]
        lib.ref_gen_eq1.argtypes = [ctypes.c_int, _c_size, _c_size, ctypes.c_uint64, _dp]
        lib.ref_split.argtypes = [ctypes.c_int, _c_size, _c_size, _dp, ctypes.c_int,
                                  ctypes.c_int, _dp, _dp]
        lib.ref_backend_gemm.argtypes = [_c_size, _c_size, _c_size, _dp, _dp, _dp]
        lib.ref_ozaki_gemm.argtypes = [ctypes.c_int, _c_size, _c_size, _c_size, _dp, _dp,
                                       ctypes.c_int, ctypes.c_double, _dp, _dp]
        lib.ref_gemm_simple.argtypes = [ctypes.c_int, _c_size, _c_size, _c_size, _dp, _dp, _dp]
        lib.ref_mf_add_double.argtypes = [ctypes.c_int, _c_size, _dp, _dp, _dp]
        lib.ref_split_shift_bits.argtypes = [_c_size]
        lib.ref_lu_update.argtypes = [ctypes.c_int, _c_size, _c_size, _c_size, _dp, _dp, _dp,
                                      ctypes.c_int]
        lib.ref_exponent_ceil_log2.argtypes = [ctypes.c_double]
        lib.ref_mpmat_write.argtypes = [ctypes.c_char_p, ctypes.c_int, _c_size, _c_size, _dp]
        lib.ref_mpmat_read.argtypes = [ctypes.c_char_p, ctypes.c_int, _c_size, _c_size, _dp]
        self.lib = lib

    def mpmat_write(self, path, a):
        """The reference's write_matrix_file (src/matrix_io.cpp); a is (m, n)
        binary64 ("d") or (m, n, K).  Returns the status (4 = io_error)."""
        a = np.ascontiguousarray(a, dtype=np.float64)
        K = 1 if a.ndim == 2 else a.shape[2]
        return self.lib.ref_mpmat_write(os.fsencode(path), K, a.shape[0], a.shape[1], _ptr(a))

    def mpmat_read(self, path, K, m, n):
        """The reference's read_matrix_file<E>: (status, array)."""
        out = np.empty((m, n) if K == 1 else (m, n, K), dtype=np.float64)
        return self.lib.ref_mpmat_read(os.fsencode(path), K, m, n, _ptr(out)), out

    def set_threads(self, t: int) -> int:
        return self.lib.ref_set_threads(t)

    def gen_eq1(self, K, m, n, seed):
        out = np.empty((m, n, K), dtype=np.float64)
        st = self.lib.ref_gen_eq1(K, m, n, seed, _ptr(out))
        if st:
            raise OracleError(st, "gen_eq1")
        return out

    def split(self, K, mat, d, side):
        mat = np.ascontiguousarray(mat, dtype=np.float64)
        rows, cols = mat.shape[0], mat.shape[1]
        pieces = np.zeros((max(d, 1), rows, cols), dtype=np.float64)
        resid = np.empty_like(mat)
        st = self.lib.ref_split(K, rows, cols, _ptr(mat), d, side, _ptr(pieces), _ptr(resid))
        if st:
            raise OracleError(st, "split")
        return pieces, resid

    def backend_gemm(self, a, b):
        a = np.ascontiguousarray(a, dtype=np.float64)
        b = np.ascontiguousarray(b, dtype=np.float64)
        c = np.empty((a.shape[0], b.shape[1]), dtype=np.float64)
        st = self.lib.ref_backend_gemm(a.shape[0], a.shape[1], b.shape[1], _ptr(a), _ptr(b),
                                       _ptr(c))
        if st:
            raise OracleError(st, "backend_gemm")
        return c

    def ozaki_gemm(self, K, a, b, d, drop=0.0, prof=None):
        a = np.ascontiguousarray(a, dtype=np.float64)
        b = np.ascontiguousarray(b, dtype=np.float64)
        m, l, n = a.shape[0], a.shape[1], b.shape[1]
        c = np.zeros((m, n, K), dtype=np.float64)
        p = np.zeros(4, dtype=np.float64)
        st = self.lib.ref_ozaki_gemm(K, m, l, n, _ptr(a), _ptr(b), d, drop, _ptr(c), _ptr(p))
        if st:
            raise OracleError(st, "ozaki_gemm")
        if prof is not None:
            prof[:] = p
        return c

    def gemm_simple(self, K, a, b):
        a = np.ascontiguousarray(a, dtype=np.float64)
        b = np.ascontiguousarray(b, dtype=np.float64)
        c = np.zeros((a.shape[0], b.shape[1], K), dtype=np.float64)
        st = self.lib.ref_gemm_simple(K, a.shape[0], a.shape[1], b.shape[1], _ptr(a), _ptr(b),
                                      _ptr(c))
        if st:
            raise OracleError(st, "gemm_simple")
        return c

    def mf_add_double(self, K, x, y):
        x = np.ascontiguousarray(x, dtype=np.float64).reshape(-1, K)
        y = np.ascontiguousarray(y, dtype=np.float64).reshape(-1)
        out = np.empty_like(x)
        self.lib.ref_mf_add_double(K, x.shape[0], _ptr(x), _ptr(y), _ptr(out))
        return out

    def exponent_ceil_log2(self, x):
        return self.lib.ref_exponent_ceil_log2(x)

    def lu_update(self, K, l21, u12, a22, d):
        """lu.hpp:104-124 trailing update on dense blocks (returns the new A22)."""
        l21 = np.ascontiguousarray(l21, dtype=np.float64)
        u12 = np.ascontiguousarray(u12, dtype=np.float64)
        out = np.array(a22, dtype=np.float64, copy=True, order="C")
        st = self.lib.ref_lu_update(K, l21.shape[0], l21.shape[1], u12.shape[1], _ptr(l21),
                                    _ptr(u12), _ptr(out), d)
        if st:
            raise OracleError(st, "lu_update")
        return out

    def split_shift_bits(self, inner, short_bits=53):
        assert short_bits == 53
        return self.lib.ref_split_shift_bits(inner)


def load_port() -> Port:
    if not os.path.exists(PORT_SO):
        build(ref=False)
    return Port()


def load_ref() -> Ref | None:
    """The compiled reference, or None when it was never built (no /root/reference)."""
    if not os.path.exists(REF_SO):
        if os.path.isdir(REF_SRC):
            build(ref=True)
        else:
            return None
    return Ref()


def best() -> CpuOzaki:
    """The compiled reference when available, else the port."""
    r = load_ref()
    return r if r is not None else load_port()
