"""Debug helper: locate bit-exactness mismatches of ozaki_gemm vs the CPU oracle."""
import sys

import numpy as np

import oracle
import paper_2301_09960_b200 as ozk

cpu = oracle.best()
cases = [(3, 256, 256, 256, 9), (4, 256, 256, 256, 12), (2, 256, 256, 256, 6)]
if len(sys.argv) > 1:
    cases = [tuple(int(x) for x in a.split(",")) for a in sys.argv[1:]]
for (K, m, l, n, d) in cases:
    a = cpu.gen_eq1(K, m, l, 11 + m + K)
    b = cpu.gen_eq1(K, l, n, 12 + m + K)
    want = cpu.ozaki_gemm(K, a, b, d)
    for rep in range(2):
        got, _ = ozk.ozaki_gemm(a, b, d)
        bad = (got.view(np.uint64) != want.view(np.uint64)).any(axis=2)
        idx = np.argwhere(bad)
        print(K, m, l, n, d, "rep", rep, "bad", int(bad.sum()), flush=True)
        if len(idx):
            print("  rows%64", np.unique(idx[:, 0] % 64), "rows//64", np.unique(idx[:, 0] // 64))
            print("  cols%128 (first 40)", np.unique(idx[:, 1] % 128)[:40])
            i, j = idx[0]
            rel = (got[i, j, 0] - want[i, j, 0]) / want[i, j, 0]
            print("  first", i, j, "got", got[i, j], "want", want[i, j], "rel", rel)
