"""Per-step timeline of the INT8 slice-GEMM kernel (CTA 0): builds a traced
libozk (-DOZK_I8_TRACE) under tools/_build and prints, per (tile, pair) step,
the MMA issuer's wait for TMEM and issue span and the epilogue's wait,
TMEM-drain and K-word-update durations in SM clocks.
python tools/i8_trace.py FMT N D  (run on the GPU box after a CPU-side build)."""
import ctypes
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
OUT = os.path.join(ROOT, "tools", "_build", "libozk_trace%s.so")


def build(mode=""):
    from paper_2301_09960_b200 import build as b
    out = OUT % mode
    os.makedirs(os.path.dirname(out), exist_ok=True)
    objs = []
    for src in b.SOURCES:
        obj = os.path.join(os.path.dirname(out), src.replace(".cu", ".trace.o"))
        flags = list(b.FLAGS)
        if src == "gemm_i8.cu":
            flags += ["-DOZK_I8_TRACE"] + ([f"-DOZK_I8_EPI_MODE={mode}"] if mode else [])
        subprocess.run([b.NVCC, *b.ARCH, *flags, "-c", os.path.join(b.CSRC, src), "-o", obj],
                       check=True)
        objs.append(obj)
    subprocess.run([b.NVCC, *b.ARCH, "-shared", "-cudart", "static", "-ccbin", "g++", "-o", out,
                    *objs], check=True)
    for o in objs:
        os.remove(o)


def main():
    if sys.argv[1] == "build":
        build(sys.argv[2] if len(sys.argv) > 2 else "")
        return
    import torch
    from paper_2301_09960_b200._lib import OzkProfile, load
    fmt, n, d = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
    lib = load(OUT % (sys.argv[4] if len(sys.argv) > 4 else ""))
    K = 3 if fmt == 0x103 else fmt
    dt = torch.float32 if fmt == 0x103 else torch.float64
    sh = torch.cuda.current_stream().cuda_stream
    A = torch.empty((n, n, K), dtype=dt, device="cuda")
    B = torch.empty_like(A)
    C = torch.empty_like(A)
    lib.ozk_gen_eq1_device(fmt, n, n, 1, A.data_ptr(), sh)
    lib.ozk_gen_eq1_device(fmt, n, n, 2, B.data_ptr(), sh)
    lib.ozk_set_engine(2)
    prof = OzkProfile()
    for _ in range(2):
        assert lib.ozk_ozaki_gemm_device(fmt, n, n, n, A.data_ptr(), B.data_ptr(), d, 0.0,
                                         C.data_ptr(), sh, ctypes.byref(prof)) == 0
    torch.cuda.synchronize()
    steps = 512
    buf = (ctypes.c_ulonglong * (8 * steps))()
    lib.ozk_i8_trace_read.argtypes = [ctypes.c_void_p, ctypes.c_int]
    assert lib.ozk_i8_trace_read(buf, steps) == 0
    t = [[buf[8 * s + j] for j in range(8)] for s in range(steps)]
    t0 = t[0][0]
    print(f"fmt={fmt} n={n} D={d} gemm {prof.product_seconds*1e3:.2f} ms")
    print("step  mma_wait  mma_issue (of which operand wait) | epi_wait  epilogue  - | step_period")
    acc = [0] * 7
    cnt = 0
    for s in range(1, steps):
        a = t[s]
        if a[6] == 0 or a[0] == 0:
            break
        row = (a[1] - a[0], a[2] - a[1], a[7], a[4] - a[3], a[5] - a[4], a[6] - a[5],
               a[4] - t[s - 1][4])
        if s < 8 or s % 100 == 0:
            print(f"{s:4d} {row[0]:9d} {row[1]:10d} {row[2]:10d} | {row[3]:8d} {row[4]:6d} "
                  f"{row[5]:6d} | {row[6]:8d}")
        if s >= 5:
            acc = [x + y for x, y in zip(acc, row)]
            cnt += 1
    if cnt:
        print("mean(steps>=5):", " ".join(f"{x/cnt:.0f}" for x in acc))


if __name__ == "__main__":
    main()
