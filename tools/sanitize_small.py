"""Smallest shapes that run every kernel of the hot path once, for
compute-sanitizer (one --tool per gpurun call):

    compute-sanitizer --tool racecheck python tools/sanitize_small.py
    compute-sanitizer --tool memcheck  python tools/sanitize_small.py

Kernels covered: split_rows_kernel (A rows / B columns, FP64 slices and INT8
digits), transpose_kernel, pair_gemm_kernel (DMMA, accumulate / products /
plain), pair_gemm_i8_kernel (DD drain, TD/QD two buffers, TS one digit with four
buffers, TS two digits, products hook), the generator and the accumulation
kernel.  Each result is checked bit for bit against the CPU oracle so a silent
corruption also fails the run.
"""
import ctypes
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import paper_2301_09960_b200 as ozk  # noqa: E402


def check(got, want, what):
    g = np.ascontiguousarray(got)
    w = np.ascontiguousarray(want)
    if not np.array_equal(g.view(np.uint8), w.view(np.uint8)):
        raise SystemExit(f"MISMATCH {what}")
    print("ok", what, flush=True)


def main():
    cpu = oracle.best()
    port = oracle.load_port()
    torch.cuda.set_device(0)
    # INT8 engine (l > 128): DD (drain), TD, QD; 2-CTA clusters with multicast
    for K, m, l, n, d in ((2, 130, 300, 260, 4), (3, 100, 260, 140, 5), (4, 50, 200, 129, 6)):
        a = cpu.gen_eq1(K, m, l, 5 + K)
        b = cpu.gen_eq1(K, l, n, 6 + K)
        got, prof = ozk.ozaki_gemm(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda(), d)
        assert prof.engine == "int8"
        check(got.cpu().numpy(), cpu.ozaki_gemm(K, a, b, d), f"int8 K={K}")
    # DMMA engine (l <= 128) and the host path (pageable staging)
    a = cpu.gen_eq1(3, 70, 96, 11)
    b = cpu.gen_eq1(3, 96, 80, 12)
    got, prof = ozk.ozaki_gemm(a, b, 6)
    assert prof.engine == "dmma"
    check(got, cpu.ozaki_gemm(3, a, b, 6), "dmma K=3 (host buffers)")
    # TS: one digit (l > 1024, 4 TMEM buffers) and two digits
    for l in (1100, 300):
        ta = port.gen_eq1_ts(40, l, 3)
        tb = port.gen_eq1_ts(l, 50, 4)
        got, _ = ozk.ozaki_gemm(torch.from_numpy(ta).cuda(), torch.from_numpy(tb).cuda(), 8)
        check(got.cpu().numpy(), port.ozaki_gemm_ts(ta, tb, 8), f"ts l={l}")
    # split with residual (both sides), backend GEMM, accumulate
    mm = cpu.gen_eq1(4, 33, 40, 21)
    for side in (0, 1):
        s = ozk.split_matrix(mm, 5, ozk.SplitSide(side))
        p, r = cpu.split(4, mm, 5, side)
        check(np.stack(s.pieces), p, f"split side={side}")
        check(s.residual, r, f"residual side={side}")
    pa, _ = cpu.split(2, cpu.gen_eq1(2, 20, 30, 1), 3, 0)
    pb, _ = cpu.split(2, cpu.gen_eq1(2, 30, 10, 2), 3, 1)
    check(ozk.gpu_backend()(pa[0], pb[1]), cpu.backend_gemm(pa[0], pb[1]), "backend gemm")
    # INT8 products hook
    K, m, l, n, d = 3, 60, 300, 70, 3
    a = cpu.gen_eq1(K, m, l, 31)
    b = cpu.gen_eq1(K, l, n, 32)
    A, B = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
    sh = torch.cuda.current_stream().cuda_stream
    ld8 = (l + 15) // 16 * 16
    dig, ex = [], []
    for side, M, rows in ((0, A, m), (1, B, n)):
        dg = torch.zeros((d, 3, rows, ld8), dtype=torch.int8, device="cuda")
        eg = torch.zeros((d, rows), dtype=torch.int32, device="cuda")
        assert ozk.lib.ozk_split_digits_device(K, M.shape[0], M.shape[1], M.shape[1],
                                               M.data_ptr(), d, side, dg.data_ptr(), ld8, rows,
                                               eg.data_ptr(), None, sh) == 0
        dig.append(dg)
        ex.append(eg)
    pairs = [(x, y) for x in range(d) for y in range(d - x)]
    flat = (ctypes.c_int * (2 * len(pairs)))(*[v for p in pairs for v in p])
    prods = torch.empty((len(pairs), m, n), dtype=torch.float64, device="cuda")
    assert ozk.lib.ozk_pair_products_digits_device(K, m, l, n, dig[0].data_ptr(),
                                                   ex[0].data_ptr(), m, dig[1].data_ptr(),
                                                   ex[1].data_ptr(), n, ld8, d, flat, len(pairs),
                                                   prods.data_ptr(), sh) == 0
    sp, _ = cpu.split(K, a, d, 0)
    sq, _ = cpu.split(K, b, d, 1)
    check(prods.cpu().numpy(), np.stack([port.exact_dgemm(sp[x], sq[y])[0] for x, y in pairs]),
          "int8 products hook")
    print("sanitize_small done", flush=True)


if __name__ == "__main__":
    main()
