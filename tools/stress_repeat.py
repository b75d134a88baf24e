"""Repeat-run stress of the slice GEMMs at production shapes (multi-wave grids,
wave pacing, TMA rings, TMEM double buffers, 2-CTA multicast): every repeat of
the same GEMM must give the same bits, alternately with poisoned scratch
($OZK_POISON_SCRATCH=1: 0xFF-filled allocations), and one sampled block is
checked against the reference.  compute-sanitizer is closed on this GPU pool;
the round-1 ring race was found exactly this way (repeat-run differences).

python tools/stress_repeat.py [reps] > profiles/r02_stress_repeat.log"""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402  (checker only)
from paper_2301_09960_b200._lib import load  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
lib = load()
ref = oracle.best()
sh = torch.cuda.current_stream().cuda_stream
# (name, format code, words, n, D, engine: 0 auto / 1 dmma / 2 int8)
cases = [("DD", 2, 2, 8192, 6, 2), ("TD", 3, 3, 8192, 9, 2), ("QD", 4, 4, 8192, 12, 2),
         ("TS", 0x103, 3, 8192, 15, 2), ("TD", 3, 3, 3000, 9, 1), ("DD", 2, 2, 4100, 40, 2)]
bad = 0
for name, code, K, n, d, eng in cases:
    dt = torch.float32 if code == 0x103 else torch.float64
    ha = torch.empty((n, n, K), dtype=dt)
    hb = torch.empty_like(ha)
    assert lib.ozk_gen_eq1(code, n, n, 11, ha.data_ptr(), 0) == 0
    assert lib.ozk_gen_eq1(code, n, n, 12, hb.data_ptr(), 0) == 0
    A, B = ha.cuda(), hb.cuda()
    C = torch.empty_like(A)
    first = None
    lib.ozk_set_engine(eng)
    t0 = time.perf_counter()
    for r in range(reps):
        os.environ["OZK_POISON_SCRATCH"] = "1" if r % 2 else "0"
        C.fill_(float("nan"))
        st = lib.ozk_ozaki_gemm_device(code, n, n, n, A.data_ptr(), B.data_ptr(), d, 0.0,
                                       C.data_ptr(), sh, None)
        assert st == 0, lib.ozk_last_error()
        torch.cuda.synchronize()
        if first is None:
            first = C.clone()
        elif not torch.equal(C.view(torch.int64 if dt == torch.float64 else torch.int32),
                             first.view(torch.int64 if dt == torch.float64 else torch.int32)):
            bad += 1
            print(f"{name} n={n} D={d} engine={eng}: repeat {r} differs", flush=True)
    t_rep = time.perf_counter() - t0
    os.environ["OZK_POISON_SCRATCH"] = "0"
    lib.ozk_set_engine(0)
    # one 256 x 256 block of the result against the reference on the same bytes
    rows = cols = 256
    a = np.ascontiguousarray(ha[:rows].numpy())
    b = np.ascontiguousarray(hb[:, :cols].numpy())
    if code == 0x103:
        want = oracle.load_port().ozaki_gemm_ts(a, b, d)
    else:
        want = ref.ozaki_gemm(K, a, b, d)
    got = first[:rows, :cols].cpu().numpy()
    ok = np.array_equal(got.view(np.uint32 if code == 0x103 else np.uint64),
                        want.view(np.uint32 if code == 0x103 else np.uint64))
    bad += 0 if ok else 1
    print(f"{name} n={n} D={d} engine={'int8' if eng == 2 else 'dmma'}: {reps} repeats "
          f"({t_rep:.1f} s, half with poisoned scratch) identical; "
          f"block vs reference {'bit-exact' if ok else 'DIFFERS'}", flush=True)
    del A, B, C, first
    torch.cuda.empty_cache()
print("FAILURES:", bad)
sys.exit(1 if bad else 0)
