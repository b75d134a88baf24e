"""Pageable vs pinned host buffers through ozk_ozaki_gemm (TD n=8192 D=9):
e2e ms per call for staging thread counts (OZK_STAGING_THREADS) and with the
staging off (OZK_PAGEABLE_STAGING=0).  python tools/staging_sweep.py [n] [reps]"""
import ctypes
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2301_09960_b200 import lib  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 4
K, d = 3, 9
ha = torch.empty((n, n, K), dtype=torch.float64, pin_memory=True)
hb = torch.empty_like(ha).pin_memory()
hc = torch.empty_like(ha).pin_memory()
assert lib.ozk_gen_eq1(K, n, n, 1, ha.data_ptr(), 0) == 0
assert lib.ozk_gen_eq1(K, n, n, 2, hb.data_ptr(), 0) == 0
pa, pb = np.array(ha.numpy()), np.array(hb.numpy())
pc = np.zeros_like(pa)


def run(a, b, c):
    st = lib.ozk_ozaki_gemm(K, n, n, n, a, b, d, 0.0, c, None)
    assert st == 0, lib.ozk_last_error()
    best = None
    for _ in range(reps):
        t0 = time.perf_counter()
        lib.ozk_ozaki_gemm(K, n, n, n, a, b, d, 0.0, c, None)
        dt = time.perf_counter() - t0
        best = dt if best is None else min(best, dt)
    return best * 1e3


print(f"pinned: {run(ha.data_ptr(), hb.data_ptr(), hc.data_ptr()):.1f} ms", flush=True)
if "--nt" in sys.argv:  # streaming-store copies on / off, default thread counts
    for nt in ["1", "0", "1", "0"]:
        os.environ["OZK_STAGING_NT"] = nt
        r = run(pa.ctypes.data, pb.ctypes.data, pc.ctypes.data)
        print(f"pageable staged, OZK_STAGING_NT={nt}: {r:.1f} ms", flush=True)
    assert np.array_equal(pc.view(np.uint64), hc.numpy().view(np.uint64))
    sys.exit(0)
for th in ["4,2", "4,4", "8,4", "8,8", "12,4", "16,8", "6,6"]:
    os.environ["OZK_STAGING_THREADS"] = th
    print(f"pageable staged threads {th}: {run(pa.ctypes.data, pb.ctypes.data, pc.ctypes.data):.1f} ms",
          flush=True)
os.environ["OZK_PAGEABLE_STAGING"] = "0"
print(f"pageable, staging off: {run(pa.ctypes.data, pb.ctypes.data, pc.ctypes.data):.1f} ms",
      flush=True)
