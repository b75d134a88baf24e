"""A/B timing of experimental libozk builds (INT8 engine), n=8192: python tools/variants_bench.py LIB..."""
import ctypes
import statistics
import sys

import torch

sys.path.insert(0, ".")
from paper_2301_09960_b200._lib import OzkProfile, load  # noqa: E402

n = 8192
sh = torch.cuda.current_stream().cuda_stream
args = sys.argv[1:]
fmts = ((2, 6), (3, 9), (4, 12))
if args and args[0].startswith("--fmts="):  # e.g. --fmts=3:9,259:15 (259 = TS)
    fmts = tuple(tuple(int(x) for x in f.split(":")) for f in args[0][7:].split(","))
    args = args[1:]
libs = [(p, load(p)) for p in args]
for fmt, d in fmts:
    K = 3 if fmt == 0x103 else fmt
    dt = torch.float32 if fmt == 0x103 else torch.float64
    A = torch.empty((n, n, K), dtype=dt)
    B = torch.empty_like(A)
    libs[0][1].ozk_gen_eq1(fmt, n, n, 1, A.data_ptr(), 0)  # the reference's inputs
    libs[0][1].ozk_gen_eq1(fmt, n, n, 2, B.data_ptr(), 0)
    A, B = A.cuda(), B.cuda()
    C = torch.empty_like(A)
    ref = None
    for path, lib in libs:
        lib.ozk_set_engine(2)
        prof = OzkProfile()
        ts, tsp = [], []
        for it in range(3):
            assert lib.ozk_ozaki_gemm_device(fmt, n, n, n, A.data_ptr(), B.data_ptr(), d, 0.0,
                                             C.data_ptr(), sh, ctypes.byref(prof)) == 0
            if it:
                ts.append(prof.product_seconds)
                tsp.append(prof.split_seconds)
        same = ""
        if ref is None:
            ref = C.clone()
        else:
            same = " (bit-identical)" if torch.equal(ref.view(torch.int32), C.view(torch.int32)) \
                else " DIFFERS"
        print(f"K={fmt} {path.split('/')[-1]}: slice GEMM {statistics.median(ts)*1e3:.1f} ms, "
              f"split {statistics.median(tsp)*1e3:.1f} ms{same}",
              flush=True)
    del A, B, C, ref
