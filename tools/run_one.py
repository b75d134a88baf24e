"""Run one Ozaki GEMM (for profiling): python tools/run_one.py FMT N D ENGINE [REPS]."""
import ctypes
import sys

import torch

sys.path.insert(0, ".")
import os  # noqa: E402

from paper_2301_09960_b200._lib import OzkProfile, load  # noqa: E402

lib = load(os.environ["OZK_LIB"]) if os.environ.get("OZK_LIB") else load()

fmt, n, d = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
eng = {"auto": 0, "dmma": 1, "int8": 2}[sys.argv[4]]
reps = int(sys.argv[5]) if len(sys.argv) > 5 else 2
lib.ozk_set_engine(eng)
sh = torch.cuda.current_stream().cuda_stream
K = 3 if fmt == 0x103 else fmt
dt = torch.float32 if fmt == 0x103 else torch.float64
A = torch.empty((n, n, K), dtype=dt, device="cuda")
B = torch.empty_like(A)
C = torch.empty_like(A)
lib.ozk_gen_eq1_device(fmt, n, n, 1, A.data_ptr(), sh)
lib.ozk_gen_eq1_device(fmt, n, n, 2, B.data_ptr(), sh)
prof = OzkProfile()
for _ in range(reps):
    assert lib.ozk_ozaki_gemm_device(fmt, n, n, n, A.data_ptr(), B.data_ptr(), d, 0.0,
                                     C.data_ptr(), sh, ctypes.byref(prof)) == 0
print(f"fmt={fmt} n={n} D={d} engine={prof.engine} gemm {prof.product_seconds*1e3:.2f} ms "
      f"split {prof.split_seconds*1e3:.2f} ms")
