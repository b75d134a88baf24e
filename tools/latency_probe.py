"""Per-call latency of ozk_ozaki_gemm_device / ozk_ozaki_gemm (pageable numpy
buffers) at small sizes: python tools/latency_probe.py (profiles/r02_call_latency.log)."""
import sys, time, torch, numpy as np
sys.path.insert(0, '.')
from paper_2301_09960_b200._lib import load
lib = load()
sh = torch.cuda.current_stream().cuda_stream
for K, n, d in ((2, 64, 6), (2, 256, 6), (3, 512, 9), (2, 1024, 6)):
    A = torch.randn(n, n, K, dtype=torch.float64, device='cuda'); A[..., 1:] = 0
    B = torch.randn(n, n, K, dtype=torch.float64, device='cuda'); B[..., 1:] = 0
    C = torch.empty_like(A)
    for _ in range(5): lib.ozk_ozaki_gemm_device(K, n, n, n, A.data_ptr(), B.data_ptr(), d, 0.0, C.data_ptr(), sh, None)
    torch.cuda.synchronize(); t = time.perf_counter(); R = 100
    for _ in range(R): lib.ozk_ozaki_gemm_device(K, n, n, n, A.data_ptr(), B.data_ptr(), d, 0.0, C.data_ptr(), sh, None)
    torch.cuda.synchronize(); dt = (time.perf_counter() - t) / R
    ha, hb, hc = A.cpu().numpy(), B.cpu().numpy(), np.empty((n, n, K))
    for _ in range(3): lib.ozk_ozaki_gemm(K, n, n, n, ha.ctypes.data, hb.ctypes.data, d, 0.0, hc.ctypes.data, None)
    t = time.perf_counter()
    for _ in range(20): lib.ozk_ozaki_gemm(K, n, n, n, ha.ctypes.data, hb.ctypes.data, d, 0.0, hc.ctypes.data, None)
    dh = (time.perf_counter() - t) / 20
    print(f"K={K} n={n} D={d}: device call {dt*1e3:.3f} ms, host call {dh*1e3:.3f} ms", flush=True)
