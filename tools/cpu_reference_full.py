"""Full-size CPU reference timings on the GPU box's host cores (one-off, recorded
under profiles/): the reference's ozaki_gemm<K> at the headline configuration
(n = 8192, reference_backend(), all host threads, OMP_PROC_BIND=close) and its
direct multi-component GEMM gemm_simple<K> (gemm.hpp:15-31) at n = 256/512/1024,
extrapolated to n = 8192 as n^3.

Also times bench.py's sampled estimate on the SAME input bytes (an r x n . n x r
sub-GEMM with per-phase scaling) so the estimate can be checked against the
full-size run.  Protocol as the reference's gemm_bench (bench.cpp:121-157):
inputs gen_matrix_eq1<K>(n, n, seed) and (n, n, seed + 1), best of reps, phase
times from the best rep.

    python tools/cpu_reference_full.py [--formats td] [--n 8192] [--out FILE]
"""
from __future__ import annotations

import argparse
import json
import os
import platform
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

HEADLINE_D = {2: 6, 3: 9, 4: 12}
NAMES = {"dd": 2, "td": 3, "qd": 4}


def host_info():
    info = {"nproc": os.cpu_count(), "platform": platform.platform()}
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True).stdout
        for line in out.splitlines():
            k, _, v = line.partition(":")
            if k.strip() in ("Model name", "Socket(s)", "Core(s) per socket",
                             "Thread(s) per core", "NUMA node(s)", "CPU(s)", "L3 cache"):
                info[k.strip()] = v.strip()
    except OSError:
        pass
    try:
        for line in open("/proc/meminfo"):
            if line.startswith(("MemTotal", "MemAvailable")):
                k, v = line.split(":")
                info[k] = v.strip()
    except OSError:
        pass
    info["OMP_PROC_BIND"] = os.environ.get("OMP_PROC_BIND")
    info["OMP_PLACES"] = os.environ.get("OMP_PLACES")
    return info


def mem_available_gib():
    for line in open("/proc/meminfo"):
        if line.startswith("MemAvailable"):
            return int(line.split()[1]) / 2**20
    return 0.0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--formats", default="td")
    ap.add_argument("--n", type=int, default=8192)
    ap.add_argument("--sample", type=int, default=1024)
    ap.add_argument("--simple-n", default="256,512")
    ap.add_argument("--skip-full", action="store_true")
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "cpu_reference_full.json"))
    args = ap.parse_args()
    os.environ.setdefault("OMP_PROC_BIND", "close")
    import numpy as np

    import oracle
    ref = oracle.load_ref()
    if ref is None:
        print("oracle/_ref missing", file=sys.stderr)
        return 1
    threads = ref.set_threads(os.cpu_count() or 1)
    res = {"host": host_info(), "threads": threads, "results": []}

    def dump():
        os.makedirs(os.path.dirname(args.out), exist_ok=True)
        with open(args.out, "w") as f:
            json.dump(res, f, indent=1)

    for fmt in args.formats.split(","):
        K = NAMES[fmt]
        d = HEADLINE_D[K]
        n = args.n
        # direct gemm_simple<K> at small n, extrapolated as n^3
        for ns in [int(x) for x in args.simple_n.split(",") if x]:
            a = ref.gen_eq1(K, ns, ns, 1)
            b = ref.gen_eq1(K, ns, ns, 2)
            reps = 3 if ns <= 256 else 1
            best = None
            for _ in range(reps):
                t0 = time.perf_counter()
                ref.gemm_simple(K, a, b)
                dt = time.perf_counter() - t0
                best = dt if best is None else min(best, dt)
            rate = 2.0 * ns ** 3 / best / 1e9
            res["results"].append({"what": "gemm_simple", "format": fmt, "n": ns, "reps": reps,
                                   "seconds": best, "gflops": rate,
                                   "extrapolated_n": n,
                                   "extrapolated_seconds": best * (n / ns) ** 3})
            print(res["results"][-1], flush=True)
            dump()
        # inputs of the headline configuration, the reference generator
        t0 = time.perf_counter()
        A = ref.gen_eq1(K, n, n, 1)
        B = ref.gen_eq1(K, n, n, 2)
        tgen = time.perf_counter() - t0
        # sampled estimate on the same bytes (bench.py's cpu_baseline method)
        r = args.sample
        prof = np.zeros(4)
        t0 = time.perf_counter()
        ref.ozaki_gemm(K, A[:r], np.ascontiguousarray(B[:, :r]), d, prof=prof)
        wall = time.perf_counter() - t0
        s = n / r
        est = prof[0] * s + (prof[1] + prof[2]) * s * s
        res["results"].append({"what": "ozaki_sample", "format": fmt, "n": n, "d": d,
                               "sample": f"{r}x{n} . {n}x{r}", "split_s": prof[0],
                               "product_s": prof[1], "accumulate_s": prof[2],
                               "wall_s": wall, "estimate_full_s": est,
                               "estimate_gflops": 2.0 * n ** 3 / est / 1e9})
        print(res["results"][-1], flush=True)
        dump()
        # the full-size run, one rep (bench.cpp: 1 rep for n >= 4096 in SURVEY's protocol)
        need = (2 * 2 + 2 * d * 2 / K + (d * (d + 1) / 2) / K + 4) * n * n * K * 8 / 2**30
        avail = mem_available_gib()
        if args.skip_full or avail < 1.3 * need:
            res["results"].append({"what": "ozaki_full", "format": fmt, "skipped":
                                   f"MemAvailable {avail:.0f} GiB < 1.3 x {need:.0f} GiB"
                                   if not args.skip_full else "--skip-full"})
            dump()
            continue
        prof = np.zeros(4)
        t0 = time.perf_counter()
        ref.ozaki_gemm(K, A, B, d, prof=prof)
        wall = time.perf_counter() - t0
        res["results"].append({"what": "ozaki_full", "format": fmt, "n": n, "d": d,
                               "gen_s": tgen, "split_s": prof[0], "product_s": prof[1],
                               "accumulate_s": prof[2], "total_s": prof[3], "wall_s": wall,
                               "gflops": 2.0 * n ** 3 / prof[3] / 1e9,
                               "mem_needed_gib": need})
        print(res["results"][-1], flush=True)
        dump()
        del A, B
    dump()
    return 0


if __name__ == "__main__":
    sys.exit(main())
