"""ctypes binding of libozk.so (the C-ABI declared in include/ozk.h).

The library is the product: there is no CPU fallback.  If the shared object is
missing or fails to load, importing this module raises -- loudly -- instead of
degrading to another implementation.
"""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "lib", "libozk.so")

OZK_OK, OZK_ESHAPE, OZK_EPARAM, OZK_ECUDA, OZK_ENCCL, OZK_ENOMEM, OZK_EIO = range(7)

_sz = ctypes.c_size_t
_dp = ctypes.c_void_p  # device or host double*, passed as raw addresses
_ip = ctypes.POINTER(ctypes.c_int)


class OzkProfile(ctypes.Structure):
    _fields_ = [
        ("split_seconds", ctypes.c_double),
        ("product_seconds", ctypes.c_double),
        ("accumulate_seconds", ctypes.c_double),
        ("total_seconds", ctypes.c_double),
        ("transfer_seconds", ctypes.c_double),
        ("split_count", ctypes.c_int),
        ("pairs", ctypes.c_int),
        ("gpus", ctypes.c_int),
        ("engine", ctypes.c_int),
    ]


# name -> (restype, argtypes); mirrors include/ozk.h one to one
SIGNATURES = {
    "ozk_ozaki_gemm": (ctypes.c_int, [ctypes.c_int, _sz, _sz, _sz, _dp, _dp, ctypes.c_int,
                                      ctypes.c_double, _dp, ctypes.POINTER(OzkProfile)]),
    "ozk_ozaki_gemm_device": (ctypes.c_int, [ctypes.c_int, _sz, _sz, _sz, _dp, _dp, ctypes.c_int,
                                             ctypes.c_double, _dp, ctypes.c_void_p,
                                             ctypes.POINTER(OzkProfile)]),
    "ozk_ozaki_gemm_device_async": (ctypes.c_int, [ctypes.c_int, _sz, _sz, _sz, _dp, _dp,
                                                   ctypes.c_int, ctypes.c_double, _dp, _dp,
                                                   ctypes.c_void_p]),
    "ozk_split": (ctypes.c_int, [ctypes.c_int, _sz, _sz, _dp, ctypes.c_int, ctypes.c_int, _dp,
                                 _dp]),
    "ozk_backend_gemm": (ctypes.c_int, [_sz, _sz, _sz, _dp, _dp, _dp]),
    "ozk_backend_gemm_device": (ctypes.c_int, [_sz, _sz, _sz, _dp, _dp, _dp, ctypes.c_void_p]),
    "ozk_split_shift_bits": (ctypes.c_int, [_sz]),
    "ozk_exponent_ceil_log2": (ctypes.c_int, [ctypes.c_double]),
    "ozk_slice_ld": (_sz, [_sz]),
    "ozk_split_slices_device": (ctypes.c_int, [ctypes.c_int, _sz, _sz, _sz, _dp, ctypes.c_int,
                                               ctypes.c_int, _dp, _sz, _dp, ctypes.c_void_p]),
    "ozk_pair_list": (ctypes.c_int, [ctypes.c_int, _dp, _dp, ctypes.c_double, _ip, _ip]),
    "ozk_slices_gemm_device": (ctypes.c_int, [ctypes.c_int, _sz, _sz, _sz, _dp, _dp, _sz, _sz,
                                              _sz, ctypes.c_int, _ip, ctypes.c_int, _dp, _sz,
                                              ctypes.c_void_p]),
    "ozk_auto_split_count": (ctypes.c_int, [ctypes.c_int, _sz]),
    "ozk_auto_drop_threshold": (ctypes.c_double, [ctypes.c_int, _sz]),
    "ozk_ozaki_gemm_multi": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_void_p, _sz,
                                            _sz, _sz, ctypes.c_void_p, ctypes.c_void_p,
                                            ctypes.c_int, ctypes.c_double, ctypes.c_void_p,
                                            ctypes.c_void_p]),
    "ozk_plan_row_bands": (ctypes.c_int, [ctypes.c_int, _sz, _sz, _sz, ctypes.c_int, _sz,
                                          ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                          ctypes.c_int, ctypes.c_void_p, ctypes.c_int]),
    "ozk_int8_digits": (ctypes.c_int, [ctypes.c_int, _sz, ctypes.c_int]),
    "ozk_split_digits_device": (ctypes.c_int, [ctypes.c_int, _sz, _sz, _sz, _dp, ctypes.c_int,
                                               ctypes.c_int, _dp, _sz, _sz, _dp, _dp,
                                               ctypes.c_void_p]),
    "ozk_split_digits_device_async": (ctypes.c_int, [ctypes.c_int, _sz, _sz, _sz, _dp,
                                                     ctypes.c_int, ctypes.c_int, _dp, _sz, _sz,
                                                     _dp, _dp, _dp, ctypes.c_void_p]),
    "ozk_check_split_flag": (ctypes.c_int, [_dp, ctypes.c_void_p]),
    "ozk_digits_gemm_device_async": (ctypes.c_int, [ctypes.c_int, _sz, _sz, _sz, _dp, _dp, _sz,
                                                    _dp, _dp, _sz, _sz, ctypes.c_int, _ip,
                                                    ctypes.c_int, _dp, _sz, ctypes.c_void_p]),
    "ozk_digits_gemm_device": (ctypes.c_int, [ctypes.c_int, _sz, _sz, _sz, _dp, _dp, _sz, _dp,
                                              _dp, _sz, _sz, ctypes.c_int, _ip, ctypes.c_int,
                                              _dp, _sz, ctypes.c_void_p]),
    "ozk_mpmat_write": (ctypes.c_int, [ctypes.c_char_p, ctypes.c_int, _sz, _sz, _dp]),
    "ozk_mpmat_read_header": (ctypes.c_int, [ctypes.c_char_p, _ip, ctypes.POINTER(_sz),
                                             ctypes.POINTER(_sz)]),
    "ozk_mpmat_read": (ctypes.c_int, [ctypes.c_char_p, ctypes.c_int, _sz, _sz, _dp]),
    "ozk_pair_products_device": (ctypes.c_int, [_sz, _sz, _sz, _dp, _dp, ctypes.c_int, _ip,
                                                ctypes.c_int, _dp, ctypes.c_void_p]),
    "ozk_pair_products_digits_device": (ctypes.c_int, [ctypes.c_int, _sz, _sz, _sz, _dp, _dp, _sz,
                                                       _dp, _dp, _sz, _sz, ctypes.c_int, _ip,
                                                       ctypes.c_int, _dp, ctypes.c_void_p]),
    "ozk_gen_eq1": (ctypes.c_int, [ctypes.c_int, _sz, _sz, ctypes.c_uint64, _dp, ctypes.c_int]),
    "ozk_gen_spread": (ctypes.c_int, [ctypes.c_int, _sz, _sz, ctypes.c_uint64, ctypes.c_int, _dp,
                                      ctypes.c_int]),
    "ozk_gen_eq1_device": (ctypes.c_int, [ctypes.c_int, _sz, _sz, ctypes.c_uint64, _dp,
                                          ctypes.c_void_p]),
    "ozk_gen_spread_device": (ctypes.c_int, [ctypes.c_int, _sz, _sz, ctypes.c_uint64,
                                             ctypes.c_int, _dp, ctypes.c_void_p]),
    "ozk_lu_trailing_update": (ctypes.c_int, [ctypes.c_int, _sz, _sz, _sz, _dp, _sz, _dp, _sz,
                                              _dp, _sz, ctypes.c_int]),
    "ozk_lu_trailing_update_device": (ctypes.c_int, [ctypes.c_int, _sz, _sz, _sz, _dp, _sz, _dp,
                                                     _sz, _dp, _sz, ctypes.c_int,
                                                     ctypes.c_void_p]),
    "ozk_direct_gemm": (ctypes.c_int, [ctypes.c_int, _sz, _sz, _sz, _dp, _dp, _dp]),
    "ozk_direct_gemm_device": (ctypes.c_int, [ctypes.c_int, _sz, _sz, _sz, _dp, _dp, _dp,
                                              ctypes.c_void_p]),
    "ozk_ts_direct_gemm": (ctypes.c_int, [_sz, _sz, _sz, _dp, _dp, _dp]),
    "ozk_ts_direct_gemm_device": (ctypes.c_int, [_sz, _sz, _sz, _dp, _dp, _dp, ctypes.c_void_p]),
    "ozk_probe_dmma_tflops": (ctypes.c_double, [ctypes.c_int, ctypes.c_void_p]),
    "ozk_probe_i8_tops": (ctypes.c_double, [ctypes.c_int, ctypes.c_void_p]),
    "ozk_set_engine": (ctypes.c_int, [ctypes.c_int]),
    "ozk_get_engine": (ctypes.c_int, []),
    "ozk_accumulate_products": (ctypes.c_int, [ctypes.c_int, _sz, _sz, ctypes.c_void_p,
                                               ctypes.c_int, _dp]),
    "ozk_accumulate_products_device": (ctypes.c_int, [ctypes.c_int, _sz, _sz, _dp, ctypes.c_int,
                                                      _dp, ctypes.c_void_p]),
    "ozk_trim_device_pool": (ctypes.c_int, []),
    "ozk_last_error": (ctypes.c_char_p, []),
    "ozk_version": (ctypes.c_int, []),
}


def load(path: str = LIB_PATH) -> ctypes.CDLL:
    if not os.path.exists(path):
        raise ImportError(
            f"libozk.so not found at {path}; build it with `python -m "
            "paper_2301_09960_b200.build` (there is no CPU fallback)")
    lib = ctypes.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = load()
