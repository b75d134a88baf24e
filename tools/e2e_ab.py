"""A/B of the host-buffer path (ozk_ozaki_gemm, pinned host A/B/C) between
libozk builds in one process: alternates the libraries, reports the median
call time per library.  python tools/e2e_ab.py FMT N D LIB...  (GPU box)"""
import ctypes
import statistics
import sys
import time

import torch

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(
    __import__("os").path.abspath(__file__))))
from paper_2301_09960_b200._lib import load  # noqa: E402


def main():
    fmt, n, d = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
    libs = [(p, load(p)) for p in sys.argv[4:]]
    K = 3 if fmt == 0x103 else fmt
    dt = torch.float32 if fmt == 0x103 else torch.float64
    sh = torch.cuda.current_stream().cuda_stream
    A = torch.empty((n, n, K), dtype=dt, device="cuda")
    B = torch.empty_like(A)
    libs[0][1].ozk_gen_eq1_device(fmt, n, n, 1, A.data_ptr(), sh)
    libs[0][1].ozk_gen_eq1_device(fmt, n, n, 2, B.data_ptr(), sh)
    hA, hB = A.cpu().pin_memory(), B.cpu().pin_memory()
    hC = [torch.empty_like(hA).pin_memory() for _ in libs]
    times = {p: [] for p, _ in libs}
    for rep in range(4):
        for i, (p, lib) in enumerate(libs):
            t = time.perf_counter()
            assert lib.ozk_ozaki_gemm(fmt, n, n, n, hA.data_ptr(), hB.data_ptr(), d, 0.0,
                                      hC[i].data_ptr(), None) == 0
            if rep:
                times[p].append(time.perf_counter() - t)
    for i, (p, _) in enumerate(libs):
        same = torch.equal(hC[i].view(torch.int64 if dt == torch.float64 else torch.int32),
                           hC[0].view(torch.int64 if dt == torch.float64 else torch.int32))
        ms = 1e3 * statistics.median(times[p])
        print(f"{p.split('/')[-1]}: {ms:.1f} ms  {2 * n ** 3 / ms / 1e6:.0f} GFLOP/s"
              f"{'' if i == 0 else (' (bit-identical)' if same else ' (DIFFERS)')}")


if __name__ == "__main__":
    main()
