"""Direct K-word GEMM (gemm_simple<MultiFloat<K>> on the GPU, csrc/direct.cu):
effective GFLOP/s (2 n^3 / t) at n (default 1024) for DD/TD/QD."""
import ctypes
import sys

import torch

sys.path.insert(0, ".")
from paper_2301_09960_b200._lib import lib  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
sh = torch.cuda.current_stream().cuda_stream
for K in (2, 3, 4):
    A = torch.empty((n, n, K), dtype=torch.float64, device="cuda")
    B = torch.empty_like(A)
    C = torch.empty_like(A)
    lib.ozk_gen_eq1_device(K, n, n, 1, A.data_ptr(), sh)
    lib.ozk_gen_eq1_device(K, n, n, 2, B.data_ptr(), sh)
    assert lib.ozk_direct_gemm_device(K, n, n, n, A.data_ptr(), B.data_ptr(), C.data_ptr(), sh) == 0
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    assert lib.ozk_direct_gemm_device(K, n, n, n, A.data_ptr(), B.data_ptr(), C.data_ptr(), sh) == 0
    e1.record()
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) * 1e-3
    print(f"direct K={K} n={n}: {t*1e3:.1f} ms = {2*n**3/t/1e9:.2f} GFLOP/s effective", flush=True)
