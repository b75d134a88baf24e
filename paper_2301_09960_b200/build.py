"""In-tree build of the CUDA library (libozk.so) for sm_100a.

nvcc only, no torch extension machinery: the library is a plain C-ABI shared
object (include/ozk.h) that Python loads with ctypes, so the same .so serves
C, C++ and Python callers.  Output: paper_2301_09960_b200/lib/libozk.so.
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB_DIR = os.path.join(HERE, "lib")
LIB = os.path.join(LIB_DIR, "libozk.so")
SOURCES = ["api.cu", "split.cu", "gemm.cu", "gen.cu", "diag.cu", "ts_direct.cu", "lu.cu", "gemm_i8.cu",
           "io.cu", "direct.cu", "accumulate.cu",
           "staging.cu"]
HOST_SOURCES = ["gen_host.cpp"]  # host-only C++ (g++, strict FP like the reference)
HEADERS = ["kword.cuh", "ozk_internal.cuh"]

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-Wall", "-Xcompiler", "-Wno-unknown-pragmas",
         "-ccbin", "g++", f"-I{os.path.join(ROOT, 'include')}"]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HOST_SOURCES + HEADERS]
    deps.append(os.path.join(ROOT, "include", "ozk.h"))
    deps.append(os.path.abspath(__file__))
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return LIB
    os.makedirs(LIB_DIR, exist_ok=True)
    objs = []
    procs = []
    for src in SOURCES:
        obj = os.path.join(LIB_DIR, src.replace(".cu", ".o"))
        cmd = [NVCC, *ARCH, *FLAGS, "-c", os.path.join(CSRC, src), "-o", obj]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        procs.append((subprocess.Popen(cmd), cmd))
        objs.append(obj)
    for src in HOST_SOURCES:
        # -ffp-contract=off: no FMA contraction, as the reference's own build
        # (proj/CMakeLists.txt:16-20); the generator must match it bit for bit
        obj = os.path.join(LIB_DIR, src.replace(".cpp", ".o"))
        cmd = ["g++", "-std=c++20", "-O2", "-ffp-contract=off", "-fPIC", "-Wall", "-Wno-unknown-pragmas", "-pthread",
               f"-I{os.path.join(ROOT, 'include')}", "-c", os.path.join(CSRC, src), "-o", obj]
        procs.append((subprocess.Popen(cmd), cmd))
        objs.append(obj)
    for p, cmd in procs:
        if p.wait() != 0:
            raise RuntimeError("nvcc failed: " + " ".join(cmd))
    link = [NVCC, *ARCH, "-shared", "-cudart", "static", "-ccbin", "g++", "-Xcompiler", "-pthread",
            "-o", LIB, *objs]
    subprocess.run(link, check=True)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
