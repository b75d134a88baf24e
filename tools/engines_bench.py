"""Time the fused Ozaki GEMM at n=8192 for DD/TD/QD under both slice-product
engines (median of 3 after 1 warm-up), reporting the slice-GEMM kernel rate."""
import ctypes
import statistics
import sys

import torch

sys.path.insert(0, ".")
from paper_2301_09960_b200._lib import OzkProfile, lib  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
sh = torch.cuda.current_stream().cuda_stream
for fmt, d in ((2, 6), (3, 9), (4, 12)):
    A = torch.empty((n, n, fmt), dtype=torch.float64, device="cuda")
    B = torch.empty_like(A)
    C = torch.empty_like(A)
    lib.ozk_gen_eq1_device(fmt, n, n, 1, A.data_ptr(), sh)
    lib.ozk_gen_eq1_device(fmt, n, n, 2, B.data_ptr(), sh)
    P = d * (d + 1) // 2
    ref = None
    for eng, name in ((1, "dmma"), (2, "int8")):
        lib.ozk_set_engine(eng)
        prof = OzkProfile()
        ts, tot = [], []
        for it in range(4):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            assert lib.ozk_ozaki_gemm_device(fmt, n, n, n, A.data_ptr(), B.data_ptr(), d, 0.0,
                                             C.data_ptr(), sh, ctypes.byref(prof)) == 0
            e1.record()
            torch.cuda.synchronize()
            if it:
                ts.append(prof.product_seconds)
                tot.append(e0.elapsed_time(e1) * 1e-3)
        t, tt = statistics.median(ts), statistics.median(tot)
        same = ""
        if ref is None:
            ref = C.clone()
        else:
            same = " bit-identical to dmma" if torch.equal(ref.view(torch.int64),
                                                           C.view(torch.int64)) else " DIFFERS"
        print(f"K={fmt} D={d} {name}: step {tt*1e3:.1f} ms = {2*n**3/tt/1e9:.1f} GFLOP/s eff; "
              f"slice GEMM {t*1e3:.1f} ms = {P*2*n**3/t/1e12:.2f} TF fp64-equiv, "
              f"{9*P*2*n**3/t/1e12:.1f} int8-TOPS-equiv{same}", flush=True)
    del A, B, C, ref
lib.ozk_set_engine(0)
