"""CSV v1 benchmark records, byte-compatible with the reference's
(proj/src/bench.cpp:21-22 header, :246-259 csv_line, :261-291 parse_csv_line,
:32-36 fmt_double), so tables from this build and from `mpmat_bench` can be
concatenated and plotted by the same tooling.

    algo,precision,n,D,K,threads,seed,reps,t_split,t_product,t_accum,t_total,max_rel_err

D (split count), K (LU panel) and max_rel_err are optional (empty fields).
Parsing mirrors the reference's std::stoul / std::stoi / std::stod calls
through the C library, so the same lines are accepted and rejected.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

HEADER = "algo,precision,n,D,K,threads,seed,reps,t_split,t_product,t_accum,t_total,max_rel_err"

_libc = ctypes.CDLL(None)
_libc.strtod.restype = ctypes.c_double
_libc.strtod.argtypes = [ctypes.c_char_p, ctypes.POINTER(ctypes.c_char_p)]
_libc.strtoull.restype = ctypes.c_ulonglong
_libc.strtoull.argtypes = [ctypes.c_char_p, ctypes.POINTER(ctypes.c_char_p), ctypes.c_int]
_libc.strtol.restype = ctypes.c_long
_libc.strtol.argtypes = [ctypes.c_char_p, ctypes.POINTER(ctypes.c_char_p), ctypes.c_int]


@dataclass
class BenchRecord:
    """bench.hpp BenchRecord."""
    algo: str = ""
    precision: str = ""
    n: int = 0
    split_count: int | None = None
    panel: int | None = None
    threads: int = 1
    seed: int = 0
    reps: int = 1
    t_split: float = 0.0
    t_product: float = 0.0
    t_accum: float = 0.0
    t_total: float = 0.0
    max_rel_err: float | None = None


def fmt_double(v: float) -> str:
    """bench.cpp:32-36: snprintf("%.17g")."""
    return "%.17g" % v


def csv_line(r: BenchRecord) -> str:
    """bench.cpp:246-259."""
    return ",".join([
        r.algo, r.precision, str(r.n),
        "" if r.split_count is None else str(r.split_count),
        "" if r.panel is None else str(r.panel),
        str(r.threads), str(r.seed), str(r.reps),
        fmt_double(r.t_split), fmt_double(r.t_product), fmt_double(r.t_accum),
        fmt_double(r.t_total),
        "" if r.max_rel_err is None else fmt_double(r.max_rel_err),
    ])


def _conv(fn, text: str, *base):
    """std::sto*: leading-prefix conversion; no digits consumed -> exception
    (ValueError here, None from parse_csv_line)."""
    buf = ctypes.create_string_buffer(text.encode())
    end = ctypes.c_char_p()
    v = fn(ctypes.cast(buf, ctypes.c_char_p), ctypes.byref(end), *base)
    if ctypes.cast(end, ctypes.c_void_p).value == ctypes.addressof(buf):
        raise ValueError(text)
    return v


def parse_csv_line(line: str) -> BenchRecord | None:
    """bench.cpp:261-291: 13 comma-separated fields, else None."""
    fields = line.split(",")
    if len(fields) != 13:
        return None
    try:
        r = BenchRecord()
        r.algo, r.precision = fields[0], fields[1]
        r.n = int(_conv(_libc.strtoull, fields[2], 10))
        if fields[3]:
            r.split_count = int(_conv(_libc.strtol, fields[3], 10))
        if fields[4]:
            r.panel = int(_conv(_libc.strtoull, fields[4], 10))
        r.threads = int(_conv(_libc.strtol, fields[5], 10))
        r.seed = int(_conv(_libc.strtoull, fields[6], 10))
        r.reps = int(_conv(_libc.strtol, fields[7], 10))
        r.t_split = _conv(_libc.strtod, fields[8])
        r.t_product = _conv(_libc.strtod, fields[9])
        r.t_accum = _conv(_libc.strtod, fields[10])
        r.t_total = _conv(_libc.strtod, fields[11])
        if fields[12]:
            r.max_rel_err = _conv(_libc.strtod, fields[12])
        return r
    except ValueError:
        return None
