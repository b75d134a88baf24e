"""B200-native Ozaki-scheme multiple-precision GEMM (DD / TD / QD / TS).

The product is ``lib/libozk.so`` (CUDA kernels for sm_100a behind the C-ABI
in ``include/ozk.h``).  ``mpmat`` mirrors the reference mpmat hot-path API on
top of it; ``sharded`` is the C block-row sharded path across GPUs (one
process per GPU, NCCL all-gather of the B digit planes); ``bench_csv`` reads
and writes the reference's CSV v1 benchmark records.
"""
from ._lib import LIB_PATH, lib  # noqa: F401  (raises if libozk.so is missing)
from .mpmat import (  # noqa: F401
    OzakiProfile,
    SplitSet,
    auto_split_policy,
    SplitSide,
    error,
    exponent_ceil_log2,
    gemm_simple,
    gen_matrix_eq1,
    get_engine,
    gpu_backend,
    io_error,
    read_matrix_file,
    lu_trailing_update,
    ozaki_gemm,
    ozaki_gemm_auto,
    ozaki_gemm_multi,
    param_error,
    shape_error,
    set_engine,
    split_matrix,
    split_shift_bits,
    ts_direct_gemm,
    write_matrix_file,
)

__all__ = [
    "OzakiProfile", "SplitSet", "SplitSide", "error", "exponent_ceil_log2", "gpu_backend",
    "ozaki_gemm", "param_error", "shape_error", "split_matrix", "split_shift_bits", "lib",
    "ts_direct_gemm", "lu_trailing_update", "set_engine", "get_engine", "io_error",
    "read_matrix_file", "write_matrix_file", "gemm_simple", "auto_split_policy",
    "ozaki_gemm_auto", "ozaki_gemm_multi", "gen_matrix_eq1",
]
