"""ozk_ozaki_gemm's host schedule (pinned buffers) for B column-block counts and
band-0 sizes ($OZK_HOST_BBLOCKS, $OZK_HOST_BAND0): median ms per call, C
checked identical.  python tools/host_schedule_sweep.py [fmt n d reps]"""
import os
import statistics
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2301_09960_b200 import lib  # noqa: E402

fmt = int(sys.argv[1]) if len(sys.argv) > 1 else 3
n = int(sys.argv[2]) if len(sys.argv) > 2 else 8192
d = int(sys.argv[3]) if len(sys.argv) > 3 else 9
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 4
K = 3 if fmt == 0x103 else fmt
dt = torch.float32 if fmt == 0x103 else torch.float64
ha = torch.empty((n, n, K), dtype=dt, pin_memory=True)
hb = torch.empty_like(ha).pin_memory()
hc = torch.empty_like(ha).pin_memory()
assert lib.ozk_gen_eq1(fmt, n, n, 1, ha.data_ptr(), 0) == 0
assert lib.ozk_gen_eq1(fmt, n, n, 2, hb.data_ptr(), 0) == 0
ref = None
settings = [("8", "", "0"), ("8", "", "2"), ("8", "", "4"), ("8", "", "6"), ("8", "", "8"),
            ("4", "", "4"), ("16", "", "8"), ("8", "", "0")]
for bb, b0, head in settings:
    os.environ["OZK_HOST_BBLOCKS"] = bb
    os.environ["OZK_HOST_HEAD"] = head
    if b0:
        os.environ["OZK_HOST_BAND0"] = b0
    else:
        os.environ.pop("OZK_HOST_BAND0", None)
    ts = []
    for r in range(reps + 1):
        t0 = time.perf_counter()
        assert lib.ozk_ozaki_gemm(fmt, n, n, n, ha.data_ptr(), hb.data_ptr(), d, 0.0,
                                  hc.data_ptr(), None) == 0
        if r:
            ts.append(time.perf_counter() - t0)
    iv = hc.view(torch.int32)
    same = "" if ref is None else (" identical" if torch.equal(iv, ref) else " DIFFERS")
    if ref is None:
        ref = iv.clone()
    ms = 1e3 * statistics.median(ts)
    print(f"bblocks={bb} band0={b0 or 'planner'} head={head}: {ms:.1f} ms {2 * n ** 3 / ms / 1e6:.0f} "
          f"GFLOP/s{same}", flush=True)
