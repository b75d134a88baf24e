"""TS n=8192 (config 4): Ozaki on both engines vs the direct TS GEMM kernel."""
import ctypes
import sys

import torch

sys.path.insert(0, ".")
from paper_2301_09960_b200._lib import OzkProfile, lib  # noqa: E402

n, d = 8192, 15
sh = torch.cuda.current_stream().cuda_stream
A = torch.empty((n, n, 3), dtype=torch.float32, device="cuda")
B = torch.empty_like(A)
C = torch.empty_like(A)
lib.ozk_gen_eq1_device(0x103, n, n, 1, A.data_ptr(), sh)
lib.ozk_gen_eq1_device(0x103, n, n, 2, B.data_ptr(), sh)
ref = None
for eng, name in ((1, "dmma"), (2, "int8")):
    lib.ozk_set_engine(eng)
    prof = OzkProfile()
    for it in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        assert lib.ozk_ozaki_gemm_device(0x103, n, n, n, A.data_ptr(), B.data_ptr(), d, 0.0,
                                         C.data_ptr(), sh, ctypes.byref(prof)) == 0
        e1.record()
        torch.cuda.synchronize()
    t = e0.elapsed_time(e1) * 1e-3
    same = ""
    if ref is None:
        ref = C.clone()
    else:
        same = " bit-identical" if torch.equal(ref.view(torch.int32), C.view(torch.int32)) else " DIFFERS"
    print(f"TS D={d} {name}: {t*1e3:.1f} ms = {2*n**3/t/1e9:.1f} GFLOP/s eff, slice GEMM "
          f"{prof.product_seconds*1e3:.1f} ms{same}", flush=True)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
lib.ozk_ts_direct_gemm_device(n, n, n, A.data_ptr(), B.data_ptr(), C.data_ptr(), sh)
e0.record()
lib.ozk_ts_direct_gemm_device(n, n, n, A.data_ptr(), B.data_ptr(), C.data_ptr(), sh)
e1.record()
torch.cuda.synchronize()
t = e0.elapsed_time(e1) * 1e-3
print(f"direct TS GEMM: {t*1e3:.1f} ms = {2*n**3/t/1e9:.1f} GFLOP/s", flush=True)
lib.ozk_set_engine(0)
