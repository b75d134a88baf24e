"""Python mirror of the reference mpmat hot-path API, running on the B200 library.

Names, argument meaning and error behaviour follow the reference C++ library
(paths relative to /root/reference/proj/include/mpmat/):

=====================================  =====================================
this module                            reference
=====================================  =====================================
``error``/``shape_error``/``param_error``  errors.hpp:7-17
``SplitSide``                          ozaki.hpp:33
``split_shift_bits``                   ozaki.hpp:43-48
``exponent_ceil_log2``                 ozaki.hpp:36-40
``SplitSet`` / ``split_matrix``        ozaki.hpp:59-67 / :74-147
``OzakiProfile``                       ozaki.hpp:149-167
``ozaki_gemm``                         ozaki.hpp:180-249 (returns ``(C, profile)``)
``gpu_backend`` (a ``GemmBackend``)    backend.hpp:12-20
=====================================  =====================================

A K-word matrix ``DenseMatrix<MultiFloat<K>>`` is a float64 array of shape
``(rows, cols, K)`` (its exact memory image); a triple-single (TS) matrix is a
float32 array of shape ``(rows, cols, 3)`` (TS is not in the reference; see
include/ozk.h).  numpy arrays and CPU torch
tensors go through the host-buffer C entry points; CUDA torch tensors go
through the device entry points on torch's current stream.
"""
from __future__ import annotations

import ctypes
import os
import enum
from dataclasses import dataclass, field

import numpy as np

from ._lib import (OZK_ECUDA, OZK_EIO, OZK_ENCCL, OZK_ENOMEM, OZK_EPARAM, OZK_ESHAPE, OzkProfile,
                   lib)

try:  # torch is optional for the host path
    import torch
except ImportError:  # pragma: no cover
    torch = None


class error(RuntimeError):
    """mpmat::error (errors.hpp:7-9)."""


class shape_error(error):
    """mpmat::shape_error (errors.hpp:11-13)."""


class param_error(error):
    """mpmat::param_error (errors.hpp:15-17)."""


class io_error(error):
    """mpmat::io_error (errors.hpp:23-25): MPMAT file I/O."""


class cuda_error(error):
    """Device failure (no reference counterpart: the reference is CPU-only)."""


def _raise(status: int) -> None:
    if status == 0:
        return
    msg = lib.ozk_last_error().decode(errors="replace")
    if status == OZK_ESHAPE:
        raise shape_error(msg)
    if status == OZK_EPARAM:
        raise param_error(msg)
    if status == OZK_ENOMEM:
        raise MemoryError(msg)
    if status == OZK_EIO:
        raise io_error(msg)
    if status in (OZK_ECUDA, OZK_ENCCL):
        raise cuda_error(msg)
    raise error(msg)


class SplitSide(enum.IntEnum):
    rows = 0  # left factor A
    cols = 1  # right factor B


FORMATS = {2: "dd", 3: "td", 4: "qd"}
OZK_TS = 0x103  # include/ozk.h
ENGINES = {0: "auto", 1: "dmma", 2: "int8"}


def set_engine(name: str) -> None:
    """Slice-product engine for subsequent calls: "auto", "dmma" or "int8"
    (include/ozk.h ozk_engine; results are bit-identical across engines)."""
    code = {v: k for k, v in ENGINES.items()}.get(name)
    if code is None:
        raise param_error(f"unknown engine {name!r}")
    _raise(lib.ozk_set_engine(code))


def get_engine() -> str:
    return ENGINES[lib.ozk_get_engine()]


def split_shift_bits(inner_dim: int) -> int:
    return lib.ozk_split_shift_bits(inner_dim)


def exponent_ceil_log2(x: float) -> int:
    return lib.ozk_exponent_ceil_log2(float(x))


@dataclass
class OzakiProfile:
    split_seconds: float = 0.0
    product_seconds: float = 0.0
    accumulate_seconds: float = 0.0
    split_count: int = 0
    pairs: int = 0
    transfer_seconds: float = 0.0
    engine: str = ""

    def total_seconds(self) -> float:
        return self.split_seconds + self.product_seconds + self.accumulate_seconds

    def _frac(self, v: float) -> float:
        t = self.total_seconds()
        return v / t if t > 0 else 0.0

    def split_fraction(self) -> float:
        return self._frac(self.split_seconds)

    def product_fraction(self) -> float:
        return self._frac(self.product_seconds)

    def accumulate_fraction(self) -> float:
        return self._frac(self.accumulate_seconds)

    @classmethod
    def _of(cls, p: OzkProfile) -> "OzakiProfile":
        return cls(p.split_seconds, p.product_seconds, p.accumulate_seconds, p.split_count,
                   p.pairs, p.transfer_seconds, ENGINES.get(p.engine, ""))


@dataclass
class SplitSet:
    pieces: list = field(default_factory=list)
    residual: np.ndarray | None = None
    side: SplitSide = SplitSide.rows
    split_count: int = 0
    short_bits: int = 53
    inner_dim: int = 0


def _is_cuda(x) -> bool:
    return torch is not None and isinstance(x, torch.Tensor) and x.is_cuda


def _is_f32(x) -> bool:
    if torch is not None and isinstance(x, torch.Tensor):
        return x.dtype == torch.float32
    return np.asarray(x).dtype == np.float32


def _kword_shape(x) -> tuple[int, int, int]:
    if x.ndim != 3:
        raise shape_error("K-word matrix must have shape (rows, cols, K)")
    r, c, k = (int(s) for s in x.shape)
    if _is_f32(x):
        if k != 3:
            raise param_error("binary32 words: only TS (K = 3) is supported")
        return r, c, OZK_TS
    if k not in FORMATS:
        raise param_error("K must be 2 (DD), 3 (TD) or 4 (QD)")
    return r, c, k


def _words(fmt: int) -> int:
    return 3 if fmt == OZK_TS else fmt


def _dtype(fmt: int):
    return np.float32 if fmt == OZK_TS else np.float64


def _host(x, fmt: int | None = None) -> np.ndarray:
    if torch is not None and isinstance(x, torch.Tensor):
        x = x.detach().cpu().numpy()
    dt = _dtype(fmt) if fmt is not None else (np.float32 if _is_f32(x) else np.float64)
    return np.ascontiguousarray(x, dtype=dt)


def _stream_handle() -> int:
    return torch.cuda.current_stream().cuda_stream


def _same_device(a, b, what: str):
    """Device context for a CUDA call on a and b: the library allocates on the
    current device and runs on its current stream, so make a's device current
    (and refuse operands on different devices)."""
    if a.device != b.device:
        raise param_error(f"{what}: A and B must live on the same device")
    return torch.cuda.device(a.device)


def ozaki_gemm(a, b, d: int, backend=None, drop_threshold: float = 0.0):
    """Long-precision product via the Ozaki split (ozaki.hpp:180-249).

    ``backend`` ``None`` or :func:`gpu_backend`: the slice products run on the
    B200 (exact INT8 tcgen05 digit GEMMs where they apply, else FP64 DMMA,
    fused with the accumulation; any conforming backend gives the same C,
    test_ozaki.cpp:227-233).  Any other callable ``backend(a_slice, b_slice)``
    is a caller's GemmBackend (backend.hpp:12-13) and is used as the reference
    uses it: called once per pair of the (pruned) triangular set, alpha-major
    (ozaki.hpp:223-231), with the split and the K-word accumulation
    (ozaki.hpp:235-244) on the B200.  Returns ``(C, OzakiProfile)``.
    """
    if backend is not None and not getattr(backend, "_ozk_gpu", False):
        return _ozaki_gemm_with_backend(a, b, int(d), backend, float(drop_threshold))
    m, l, ka = _kword_shape(a)
    l2, n, kb = _kword_shape(b)
    if ka != kb:
        raise param_error("ozaki_gemm: A and B must have the same format")
    if l != l2:
        raise shape_error("ozaki_gemm: inner dimensions differ")
    prof = OzkProfile()
    K = _words(ka)
    if _is_cuda(a) or _is_cuda(b):
        if not (_is_cuda(a) and _is_cuda(b)):
            raise param_error("ozaki_gemm: A and B must live on the same device")
        with _same_device(a, b, "ozaki_gemm"):
            ad, bd = a.contiguous(), b.contiguous()
            c = torch.empty((m, n, K), dtype=ad.dtype, device=a.device)
            st = lib.ozk_ozaki_gemm_device(ka, m, l, n, ad.data_ptr(), bd.data_ptr(), int(d),
                                           float(drop_threshold), c.data_ptr(), _stream_handle(),
                                           ctypes.byref(prof))
        _raise(st)
        return c, OzakiProfile._of(prof)
    ah, bh = _host(a, ka), _host(b, ka)
    c = np.empty((m, n, K), dtype=_dtype(ka))
    st = lib.ozk_ozaki_gemm(ka, m, l, n, ah.ctypes.data, bh.ctypes.data, int(d),
                            float(drop_threshold), c.ctypes.data, ctypes.byref(prof))
    _raise(st)
    return c, OzakiProfile._of(prof)


def _ozaki_gemm_with_backend(a, b, d, backend, drop):
    import time
    m, l, ka = _kword_shape(a)
    l2, n, kb = _kword_shape(b)
    if ka != kb:
        raise param_error("ozaki_gemm: A and B must have the same format")
    if l != l2:
        raise shape_error("ozaki_gemm: inner dimensions differ")
    if d < 1:
        raise param_error("ozaki_gemm: split count must be >= 1")
    if drop < 0.0:
        raise param_error("ozaki_gemm: negative drop threshold")
    t0 = time.perf_counter()
    sa = split_matrix(_host(a, ka), d, SplitSide.rows)
    sb = split_matrix(_host(b, ka), d, SplitSide.cols)
    t1 = time.perf_counter()
    amax = np.array([np.max(np.abs(p)) if p.size else 0.0 for p in sa.pieces], dtype=np.float64)
    bmax = np.array([np.max(np.abs(p)) if p.size else 0.0 for p in sb.pieces], dtype=np.float64)
    pairs = (ctypes.c_int * (2 * d * d))()
    np_ = ctypes.c_int(0)
    _raise(lib.ozk_pair_list(d, amax.ctypes.data, bmax.ctypes.data, drop, pairs,
                             ctypes.byref(np_)))
    products = []
    for p in range(np_.value):
        c = np.ascontiguousarray(backend(sa.pieces[pairs[2 * p]].astype(np.float64),
                                         sb.pieces[pairs[2 * p + 1]].astype(np.float64)),
                                 dtype=np.float64)
        if c.shape != (m, n):
            raise shape_error("ozaki_gemm: backend returned a product of the wrong shape")
        products.append(c)
    t2 = time.perf_counter()
    ptrs = (ctypes.c_void_p * max(len(products), 1))(*[c.ctypes.data for c in products])
    out = np.empty((m, n, _words(ka)), dtype=_dtype(ka))
    _raise(lib.ozk_accumulate_products(ka, m, n, ptrs, len(products), out.ctypes.data))
    t3 = time.perf_counter()
    prof = OzakiProfile(split_seconds=t1 - t0, product_seconds=t2 - t1,
                        accumulate_seconds=t3 - t2, split_count=d, pairs=len(products))
    return out, prof


def ozaki_gemm_multi(a, b, d: int, devices=None, drop_threshold: float = 0.0):
    """ozaki_gemm over several GPUs in one process (include/ozk.h
    ozk_ozaki_gemm_multi): C block rows per device, B digit planes all-gathered
    by peer copies; bit-identical to ozaki_gemm.  Host (numpy) arrays; devices:
    list of CUDA device ids (a device may repeat), default all visible ones.
    Returns (C, OzakiProfile)."""
    m, l, ka = _kword_shape(a)
    l2, n, kb = _kword_shape(b)
    if ka != kb:
        raise param_error("ozaki_gemm_multi: A and B must have the same format")
    if l != l2:
        raise shape_error("ozaki_gemm_multi: inner dimensions differ")
    if devices is None:
        import torch
        devices = list(range(torch.cuda.device_count()))
    devs = (ctypes.c_int * len(devices))(*[int(x) for x in devices])
    ah, bh = _host(a, ka), _host(b, ka)
    c = np.empty((m, n, _words(ka)), dtype=_dtype(ka))
    prof = OzkProfile()
    st = lib.ozk_ozaki_gemm_multi(ka, len(devices), devs, m, l, n, ah.ctypes.data, bh.ctypes.data,
                                  int(d), float(drop_threshold), c.ctypes.data, ctypes.byref(prof))
    _raise(st)
    return c, OzakiProfile._of(prof)


def auto_split_policy(fmt: int, inner_dim: int) -> tuple[int, float]:
    """(split_count, drop_threshold) of the automatic mode (include/ozk.h
    ozk_auto_split_count / ozk_auto_drop_threshold; not in the reference)."""
    return (int(lib.ozk_auto_split_count(fmt, inner_dim)),
            float(lib.ozk_auto_drop_threshold(fmt, inner_dim)))


def ozaki_gemm_auto(a, b):
    """ozaki_gemm with the automatic split count: enough slices for the full
    K-word significand and the reference's own pair pruning at the format's
    precision, so only the pairs that can change C are computed.  Equals the
    reference's ozaki_gemm(a, b, D, backend, drop) for the returned D, drop.
    Returns (C, OzakiProfile, D, drop)."""
    _, l, fmt = _kword_shape(a)
    d, drop = auto_split_policy(fmt, l)
    c, prof = ozaki_gemm(a, b, d, drop_threshold=drop)
    return c, prof, d, drop


def gen_matrix_eq1(fmt: int, m: int, n: int, seed: int, spread: int = 0) -> np.ndarray:
    """gen_matrix_eq1<K>(m, n, seed) (gen.hpp:20-34): the reference's input
    generator, bit for bit, on all host cores (csrc/gen_host.cpp).  fmt: K = 2,
    3, 4 or OZK_TS; spread > 0 gives the config-5 exponent-spread variant."""
    out = np.empty((m, n, _words(fmt)), dtype=_dtype(fmt))
    if spread:
        st = lib.ozk_gen_spread(fmt, m, n, seed, spread, out.ctypes.data, 0)
    else:
        st = lib.ozk_gen_eq1(fmt, m, n, seed, out.ctypes.data, 0)
    _raise(st)
    return out


def split_matrix(m, d: int, side: SplitSide) -> SplitSet:
    """split_matrix<K> (ozaki.hpp:74-147): pieces + K-word residual (host arrays)."""
    rows, cols, k = _kword_shape(m)
    mh = _host(m, k)
    dd = max(int(d), 1)
    pieces = np.zeros((dd, rows, cols), dtype=_dtype(k))
    resid = np.empty_like(mh)
    st = lib.ozk_split(k, rows, cols, mh.ctypes.data, int(d), int(side), pieces.ctypes.data,
                       resid.ctypes.data)
    _raise(st)
    return SplitSet(pieces=[pieces[i] for i in range(dd)], residual=resid, side=SplitSide(side),
                    split_count=int(d), inner_dim=cols if side == SplitSide.rows else rows,
                    short_bits=24 if k == OZK_TS else 53)


def gpu_backend():
    """A GemmBackend (backend.hpp:12-13): ``c = backend(a, b)`` on binary64 matrices."""

    def backend(a, b):
        if _is_cuda(a) and _is_cuda(b):
            ad, bd = a.contiguous(), b.contiguous()
            m, l = ad.shape
            l2, n = bd.shape
            if l != l2:
                raise shape_error("backend: inner dimensions differ")
            with _same_device(a, b, "backend"):
                c = torch.empty((m, n), dtype=torch.float64, device=a.device)
                _raise(lib.ozk_backend_gemm_device(m, l, n, ad.data_ptr(), bd.data_ptr(),
                                                   c.data_ptr(), _stream_handle()))
            return c
        ah, bh = _host(a), _host(b)
        if ah.ndim != 2 or bh.ndim != 2 or ah.shape[1] != bh.shape[0]:
            raise shape_error("backend: inner dimensions differ")
        c = np.empty((ah.shape[0], bh.shape[1]), dtype=np.float64)
        _raise(lib.ozk_backend_gemm(ah.shape[0], ah.shape[1], bh.shape[1], ah.ctypes.data,
                                    bh.ctypes.data, c.ctypes.data))
        return c

    backend._ozk_gpu = True
    return backend


def ts_direct_gemm(a, b):
    """Direct triple-single GEMM (config-4 comparator; csrc/ts_direct.cu)."""
    m, l, fa = _kword_shape(a)
    l2, n, fb = _kword_shape(b)
    if fa != OZK_TS or fb != OZK_TS:
        raise param_error("ts_direct_gemm: float32 (rows, cols, 3) TS matrices required")
    if l != l2:
        raise shape_error("ts_direct_gemm: inner dimensions differ")
    if _is_cuda(a) and _is_cuda(b):
        ad, bd = a.contiguous(), b.contiguous()
        with _same_device(a, b, "ts_direct_gemm"):
            c = torch.empty((m, n, 3), dtype=torch.float32, device=a.device)
            _raise(lib.ozk_ts_direct_gemm_device(m, l, n, ad.data_ptr(), bd.data_ptr(),
                                                 c.data_ptr(), _stream_handle()))
        return c
    ah, bh = _host(a, OZK_TS), _host(b, OZK_TS)
    c = np.empty((m, n, 3), dtype=np.float32)
    _raise(lib.ozk_ts_direct_gemm(m, l, n, ah.ctypes.data, bh.ctypes.data, c.ctypes.data))
    return c


def gemm_simple(a, b):
    """gemm_simple<MultiFloat<K>> (gemm.hpp:15-31) on the GPU, bit-identical:
    fixed k-order K-word multiply-accumulate (csrc/direct.cu).  TS inputs go
    to ts_direct_gemm."""
    m, l, fa = _kword_shape(a)
    l2, n, fb = _kword_shape(b)
    if fa != fb:
        raise param_error("gemm_simple: A and B must have the same format")
    if fa == OZK_TS:
        return ts_direct_gemm(a, b)
    if l != l2:
        raise shape_error("gemm_simple: inner dimensions differ")
    K = _words(fa)
    if _is_cuda(a) and _is_cuda(b):
        ad, bd = a.contiguous(), b.contiguous()
        with _same_device(a, b, "gemm_simple"):
            c = torch.empty((m, n, K), dtype=torch.float64, device=a.device)
            _raise(lib.ozk_direct_gemm_device(fa, m, l, n, ad.data_ptr(), bd.data_ptr(),
                                              c.data_ptr(), _stream_handle()))
        return c
    ah, bh = _host(a, fa), _host(b, fa)
    c = np.empty((m, n, K), dtype=np.float64)
    _raise(lib.ozk_direct_gemm(fa, m, l, n, ah.ctypes.data, bh.ctypes.data, c.ctypes.data))
    return c


def lu_trailing_update(a22, l21, u12, d: int = 6):
    """Blocked-LU trailing update A22 -= L21 * U12 (lu.hpp:104-124) in place on a
    host K-word array (or view with unit element stride); Ozaki product with d
    slices (GemmChoice::split_count default 6, lu.hpp:18)."""
    tm, pw, fa = _kword_shape(l21)
    pw2, tn, fb = _kword_shape(u12)
    tm2, tn2, fc = _kword_shape(a22)
    if not (fa == fb == fc) or fa == OZK_TS:
        raise param_error("lu_trailing_update: DD/TD/QD blocks of one format required")
    if pw != pw2 or tm != tm2 or tn != tn2:
        raise shape_error("lu_trailing_update: block shapes differ")
    K = _words(fa)

    def strided(x):
        x = np.asarray(x)
        if x.dtype != np.float64 or x.strides[2] != 8 or x.strides[1] != 8 * K:
            raise param_error("lu_trailing_update: float64 K-word blocks with unit element stride")
        return x, x.strides[0] // (8 * K)
    l, ldl = strided(l21)
    u, ldu = strided(u12)
    a, lda = strided(a22)
    _raise(lib.ozk_lu_trailing_update(fa, tm, pw, tn, l.ctypes.data, ldl, u.ctypes.data, ldu,
                                      a.ctypes.data, lda, int(d)))


# ---- MPMAT v1 matrix files (proj/src/matrix_io.cpp; csrc/io.cu) ------------

OZK_D = 1  # plain binary64 matrix, tag "d"
_TAGS = {OZK_D: "d", 2: "dd", 3: "td", 4: "qd", OZK_TS: "ts"}


def write_matrix_file(path: str, a) -> None:
    """write_matrix_file (matrix_io.hpp:43-46): a is (m, n) binary64 ("d"),
    (m, n, K) binary64 K-word (dd/td/qd) or (m, n, 3) binary32 (ts)."""
    x = a.detach().cpu().numpy() if torch is not None and isinstance(a, torch.Tensor) else a
    x = np.asarray(x)
    if x.ndim == 2:
        fmt, m, n = OZK_D, int(x.shape[0]), int(x.shape[1])
        x = np.ascontiguousarray(x, dtype=np.float64)
    else:
        m, n, fmt = _kword_shape(x)
        x = _host(x, fmt)
    _raise(lib.ozk_mpmat_write(os.fsencode(path), fmt, m, n, x.ctypes.data))


def read_matrix_file(path: str, tag: str | None = None) -> np.ndarray:
    """read_matrix_file<E> (matrix_io.hpp:51-52).  tag (d/dd/td/qd/ts) plays the
    role of the element type E: a file with another tag raises io_error, as
    in the reference.  Without it the file's own tag is used."""
    fmt = ctypes.c_int(0)
    m, n = ctypes.c_size_t(0), ctypes.c_size_t(0)
    _raise(lib.ozk_mpmat_read_header(os.fsencode(path), ctypes.byref(fmt), ctypes.byref(m),
                                     ctypes.byref(n)))
    want = fmt.value
    if tag is not None:
        inv = {v: k for k, v in _TAGS.items()}
        if tag not in inv:
            raise param_error(f"unknown precision tag {tag!r}")
        want = inv[tag]
    k = 1 if want == OZK_D else _words(want)
    shape = (m.value, n.value) if want == OZK_D else (m.value, n.value, k)
    out = np.empty(shape, dtype=np.float32 if want == OZK_TS else np.float64)
    _raise(lib.ozk_mpmat_read(os.fsencode(path), want, m.value, n.value, out.ctypes.data))
    return out
