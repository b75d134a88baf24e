"""Split-count sweep at n = 8192: effective GFLOP/s of
the INT8 engine for DD D=4..8, TD D=7..11, QD D=9..14 (median of 2 after a
warm-up), one JSON object per line.  python tools/d_sweep.py [n] [K:lo-hi,...]
(e.g. `4096 2:2-10` = BASELINE config 2, DD n=4096 with the split count swept)."""
import ctypes
import json
import statistics
import sys

import torch

sys.path.insert(0, ".")
from paper_2301_09960_b200._lib import OzkProfile, lib  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
sh = torch.cuda.current_stream().cuda_stream
lib.ozk_set_engine(2)
plan = ((2, range(4, 9)), (3, range(7, 12)), (4, range(9, 15)))
if len(sys.argv) > 2:
    plan = tuple((int(f.split(":")[0]), range(int(f.split(":")[1].split("-")[0]),
                                               int(f.split(":")[1].split("-")[1]) + 1))
                 for f in sys.argv[2].split(","))
for K, ds in plan:
    A = torch.empty((n, n, K), dtype=torch.float64)
    B = torch.empty_like(A)
    lib.ozk_gen_eq1(K, n, n, 1, A.data_ptr(), 0)  # the reference's inputs (bench.cpp:111-112)
    lib.ozk_gen_eq1(K, n, n, 2, B.data_ptr(), 0)
    A, B = A.cuda(), B.cuda()
    C = torch.empty_like(A)
    for d in ds:
        ts, tk = [], []
        prof = OzkProfile()
        for it in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            assert lib.ozk_ozaki_gemm_device(K, n, n, n, A.data_ptr(), B.data_ptr(), d, 0.0,
                                             C.data_ptr(), sh, ctypes.byref(prof)) == 0
            e1.record()
            torch.cuda.synchronize()
            if it:
                ts.append(e0.elapsed_time(e1) * 1e-3)
                tk.append(prof.product_seconds)
        t = statistics.median(ts)
        print(json.dumps({"format": {2: "DD", 3: "TD", 4: "QD"}[K], "n": n, "D": d,
                          "pairs": d * (d + 1) // 2, "engine": "int8",
                          "gflops_effective": round(2 * n ** 3 / t / 1e9, 1),
                          "ms_per_step": round(1e3 * t, 2),
                          "slice_gemm_ms": round(1e3 * statistics.median(tk), 2)}), flush=True)
    del A, B, C
lib.ozk_set_engine(0)
