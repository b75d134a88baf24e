"""Experiment: time the fused Ozaki GEMM for DD/TD/QD at n=8192 with the product
library and (optionally) an experimental build, several steps each."""
import ctypes
import statistics
import sys

import torch

sys.path.insert(0, ".")
from paper_2301_09960_b200._lib import SIGNATURES, OzkProfile, load  # noqa: E402

libs = {"prod": load("paper_2301_09960_b200/lib/libozk.so")}
for extra in sys.argv[1:]:
    libs[extra] = load(extra)
n = 8192
sh = torch.cuda.current_stream().cuda_stream
for fmt, d in ((2, 6), (3, 9), (4, 12)):
    A = torch.empty((n, n, fmt), dtype=torch.float64, device="cuda")
    B = torch.empty_like(A)
    C = torch.empty_like(A)
    libs["prod"].ozk_gen_eq1_device(fmt, n, n, 1, A.data_ptr(), sh)
    libs["prod"].ozk_gen_eq1_device(fmt, n, n, 2, B.data_ptr(), sh)
    P = d * (d + 1) // 2
    for name, lib in libs.items():
        prof = OzkProfile()
        ts = []
        for it in range(4):
            assert lib.ozk_ozaki_gemm_device(fmt, n, n, n, A.data_ptr(), B.data_ptr(), d, 0.0,
                                             C.data_ptr(), sh, ctypes.byref(prof)) == 0
            if it:
                ts.append(prof.product_seconds)
        t = statistics.median(ts)
        print(f"K={fmt} D={d} {name}: gemm {t*1e3:.1f} ms  {P*2*n**3/t/1e12:.2f} TF  "
              f"frac {P*2*n**3/t/1e12/37.1:.3f}  spread {min(ts)*1e3:.1f}-{max(ts)*1e3:.1f}",
              flush=True)
    del A, B, C
