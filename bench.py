#!/usr/bin/env python3
"""Benchmark of the B200 Ozaki-scheme multiple-precision GEMM (BASELINE.json metric).

One "step" = one full Ozaki GEMM C = A*B at n = 8192 (split of A and B into
FP64 slices, the P = D(D+1)/2 slice-pair DMMA GEMMs, and the fused K-word
accumulation) on device-resident synthetic Eq. (1) inputs.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--format td] [--impl ours|reference]

N > 1 runs under torchrun: C block-rows are sharded across ranks, each rank
splits its A row block and its B column block, and the B slices are
all-gathered over NCCL (paper_2301_09960_b200/sharded.py).  Rank 0 prints ONE
JSON line.  ``--impl reference`` times the reference's own CPU implementation
(oracle/_ref, the unmodified reference compiled in place; the C restatement
when that is absent) on all host cores on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
# the host CPUs this process may use, taken before torch's OpenMP runtime can
# pin the main thread (the CPU legs restore it and use all of them)
HOST_CPUS = sorted(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else None

METRIC = ("effective DD/TD/QD GEMM GFLOP/s (2n^3/t), n=8192; slice DGEMM % of FP64 peak")
DATA = ("synthetic: the reference's own inputs gen_matrix_eq1<K>(n, n, 1) and (n, n, 2) "
        "(gen.hpp:20-34, bench.cpp:111-112), generated bit-identically on the host by "
        "ozk_gen_eq1; both arms see the same bytes")
# format -> (ozk_format code, words, headline D).  DD/TD/QD: SURVEY §8d saturating D at
# l = 8192; TS (config 4): 5-bit slices at sigma_TS = 19, saturation near D = 15.
WORKLOADS = {"dd": (2, 2, 6), "td": (3, 3, 9), "qd": (4, 4, 12), "ts": (0x103, 3, 15)}
NAMES = {"dd": "DD", "td": "TD", "qd": "QD", "ts": "TS"}


def fmt_info(fmt):
    code, K, d = WORKLOADS[fmt]
    return code, K, d, (4 if fmt == "ts" else 8)
KERNELS_PER_STEP = 4  # split A, transpose B, split B, fused slice GEMM (either engine)


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=3)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--format", choices=sorted(WORKLOADS), default="td")
    p.add_argument("--n", type=int, default=8192)
    p.add_argument("--d", type=int, default=None)
    p.add_argument("--variants", default="dd,qd,ts",
                   help="other formats timed (1 step each) and reported under 'variants'")
    p.add_argument("--engine", choices=["auto", "dmma", "int8"], default="auto",
                   help="slice-product engine (bit-identical results; auto = INT8 where it "
                        "applies)")
    p.add_argument("--spread", type=int, default=0,
                   help="config 5: scale every element by 2^U[-s,s] (ill-conditioned inputs)")
    p.add_argument("--cpu-sample", type=int, default=1024,
                   help="rows/cols of the CPU baseline sub-GEMM (inner dim stays n)")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-cpu-direct", action="store_true",
                   help="skip timing the reference's direct gemm_simple<K> on the host")
    p.add_argument("--cpu-direct-n", type=int, default=256)
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-e2e-pageable", action="store_true")
    p.add_argument("--no-engine-compare", action="store_true",
                   help="skip timing the other slice-product engine (for large n, where one "
                        "DMMA step takes tens of seconds)")
    p.add_argument("--csv", default=None,
                   help="also append the headline run as a CSV v1 record (the reference's "
                        "bench table format, bench.cpp:21-22,246-259; `threads` = GPUs)")
    return p.parse_args()


def dist_env():
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


# ---------------------------------------------------------------------------
# clocks during the timed region (B200_PROFILING.md recipe)
# ---------------------------------------------------------------------------
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.path = None
        self.skip = 0

    def _lines(self):
        try:
            with open(self.path) as f:
                return sum(1 for _ in f)
        except OSError:
            return 0

    def start(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except (OSError, FileNotFoundError):
            self.proc = None
            return
        # nvidia-smi takes a while to start: wait (outside the timed region)
        # for its first line so short timed regions are sampled too, and
        # drop the lines written before the region starts
        t0 = time.monotonic()
        while self._lines() == 0 and time.monotonic() - t0 < 5.0 and self.proc.poll() is None:
            time.sleep(0.02)
        self.skip = self._lines()

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        lines = open(self.path).read().splitlines()
        if len(lines) > self.skip:
            lines = lines[self.skip:]
        else:  # the region was shorter than one sampling period: the last sample
            lines = lines[-1:]
        rows = []
        for line in lines:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                rows.append((float(parts[1]), float(parts[2]), float(parts[3]), parts[5:9]))
            except ValueError:
                continue
        os.unlink(self.path)
        if not rows:
            return None
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i, v in enumerate(r[3]) if v == "Active"})
        return {"sm_mhz": statistics.median(r[0] for r in rows), "sm_max_mhz": rows[0][1],
                "power_w_max": max(r[2] for r in rows), "samples": len(rows),
                "reasons": reasons}


# ---------------------------------------------------------------------------
# CPU arms (oracle/: the reference compiled in place, else the C restatement)
# ---------------------------------------------------------------------------
def host_cpu_info():
    """lscpu model, usable cores and OpenMP binding of the host running the CPU arm."""
    info = {"cores_usable": len(HOST_CPUS) if HOST_CPUS else os.cpu_count(), "OMP_PROC_BIND": os.environ.get("OMP_PROC_BIND"),
            "OMP_PLACES": os.environ.get("OMP_PLACES")}
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            k, _, v = line.partition(":")
            if k.strip() in ("Model name", "Socket(s)", "Core(s) per socket", "Thread(s) per core"):
                info[k.strip()] = v.strip()
    except (OSError, subprocess.SubprocessError):
        pass
    return info


def full_size_record(fmt):
    """The one-off full-size reference run on this box type (tools/cpu_reference_full.py,
    committed under profiles/), if present: validates the sampled estimate."""
    path = os.path.join(ROOT, "profiles", "cpu_reference_full_r02.json")
    if not os.path.exists(path):
        return None
    try:
        res = json.load(open(path))
    except (OSError, ValueError):
        return None
    for r in res.get("results", []):
        if r.get("what") == "ozaki_full" and r.get("format") == fmt and "total_s" in r:
            return {"n": r["n"], "d": r["d"], "total_s": round(r["total_s"], 2),
                    "gflops": round(r["gflops"], 4), "split_s": round(r["split_s"], 2),
                    "product_s": round(r["product_s"], 2),
                    "accumulate_s": round(r["accumulate_s"], 2),
                    "threads": res.get("threads"), "source": "profiles/cpu_reference_full_r02.json"}
    return None


def cpu_sample(cpu, K, d, n, r, a_rows, b_cols):
    """Reference CPU Ozaki on the r x n . n x r sub-GEMM A[:r] . B[:, :r] of the
    workload's own input bytes (same inner dimension, so the same sigma, slice
    widths, D and pair list), timed as the reference's gemm_bench does
    (bench.cpp:121-157: wall time of ozaki_gemm, phase times from its
    OzakiProfile).  The full n x n time is estimated per phase: the split
    scales with the split elements (2rn -> 2n^2: x n/r), the slice products and
    the accumulation with the C elements (r^2 -> n^2: x (n/r)^2).
    Returns (C_sub, sample wall s, estimated full-size s, profile)."""
    import numpy as np
    prof = np.zeros(4)
    t0 = time.perf_counter()
    c = cpu.ozaki_gemm(K, a_rows, b_cols, d, prof=prof) if cpu.kind == "reference" \
        else cpu.ozaki_gemm(K, a_rows, b_cols, d)
    wall = time.perf_counter() - t0
    if cpu.kind != "reference":  # the C restatement has no phase timers: all as products
        prof[:] = (0.0, wall, 0.0, wall)
    s = n / r
    est = prof[0] * s + (prof[1] + prof[2]) * s * s
    return c, wall, est, prof


def cpu_direct(cpu, K, n, nd, a, b):
    """The reference's direct multi-component GEMM gemm_simple<MultiFloat<K>>
    (gemm.hpp:15-31) on the leading nd x nd blocks of the same inputs, timed
    on all host threads and extrapolated to n as n^3 (its cost is cubic)."""
    import numpy as np
    aa = np.ascontiguousarray(a[:nd, :nd])
    bb = np.ascontiguousarray(b[:nd, :nd])
    t0 = time.perf_counter()
    cpu.gemm_simple(K, aa, bb)
    dt = time.perf_counter() - t0
    return {"n": nd, "seconds": round(dt, 4), "gflops": round(2.0 * nd ** 3 / dt / 1e9, 5),
            "extrapolated_n": n, "extrapolated_seconds": round(dt * (n / nd) ** 3, 1),
            "note": "reference gemm_simple<MultiFloat<K>> (gemm.hpp:15-31), all host threads, "
                    "extrapolated as n^3"}


def reference_inputs(cpu, K, n, r, spread):
    """The sampled blocks A[:r] and B[:, :r] of gen_matrix_eq1<K>(n, n, 1) and
    (n, n, 2) (bench.cpp:111-112 seeds), from the reference generator itself."""
    import numpy as np
    port = None
    if spread:
        import oracle
        port = oracle.load_port()
        a = port.gen_spread(K, r, n, 1, spread)  # first r rows of the stream
        b = port.gen_spread(K, n, n, 2, spread)
    else:
        a = cpu.gen_eq1(K, r, n, 1)  # the stream is row-major: rows 0..r-1 of (n, n)
        b = cpu.gen_eq1(K, n, n, 2)
    return a, np.ascontiguousarray(b[:, :r])


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    code, K, d0, _ = fmt_info(args.format)
    if args.format == "ts":
        print(json.dumps({"impl": "reference", "unavailable":
                          "TS is not implemented by the reference (SPEC.md:8)"}), flush=True)
        return 0
    import oracle
    cpu = oracle.best()
    cores = cpu.set_threads(len(HOST_CPUS or [1])) if hasattr(cpu, "set_threads") else 1
    d = args.d or d0
    n, r = args.n, min(args.cpu_sample, args.n)
    a, b = reference_inputs(cpu, K, n, r, args.spread)
    for _ in range(args.warmup):
        cpu_sample(cpu, K, d, n, r, a, b)
    walls, ests = [], []
    for _ in range(args.steps):
        _, wall, est, _ = cpu_sample(cpu, K, d, n, r, a, b)
        walls.append(wall)
        ests.append(est)
    t_full = min(ests)  # best of reps, as bench.cpp:144-152
    value = 2.0 * n ** 3 / t_full / 1e9
    sample = (f"{NAMES[args.format]} Ozaki sub-GEMM A[:{r}] . B[:, :{r}] of the n={n} inputs "
              f"(gen_matrix_eq1 seeds 1, 2), D={d}, reference ozaki_gemm<K> + "
              f"reference_backend(); full n x n time estimated per phase (split x n/r, "
              f"products + accumulation x (n/r)^2), best of {args.steps}")
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": "GFLOP/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(1e3 * statistics.mean(walls), 3), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": DATA,
        "config": config_of(args, K, d, n),
        "cpu_baseline": {"value": round(value, 4), "unit": "GFLOP/s", "cores": cores,
                         "kind": cpu.kind, "sample": sample,
                         "estimated_full_seconds": round(t_full, 2),
                         "ms_per_step_is": "wall time of one sampled sub-GEMM",
                         "host": host_cpu_info(),
                         "full_size_measured": full_size_record(args.format)},
        "e2e": {"value": round(value, 4), "unit": "GFLOP/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def config_of(args, K, d, n):
    wl = f"{NAMES[args.format]} Ozaki GEMM n={n} D={d} (BASELINE config 3)"
    if args.spread:
        wl = (f"ill-conditioned {NAMES[args.format]} Ozaki GEMM n={n} D={d}, exponent spread "
              f"+-{args.spread} (BASELINE config 5)")
    elif args.format == "ts":
        wl = f"TS Ozaki GEMM n={n} D={d} (BASELINE config 4)"
    return {"workload": wl, "spread": args.spread,
            "format": args.format, "n": n, "split_count": d, "pairs": d * (d + 1) // 2,
            "parallelism": f"C block-rows x{args.gpus}" if args.gpus > 1 else "single GPU",
            "l2": "no flush: A, B and C are each > 126 MB L2 (K*8*n^2 bytes)"}


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
ENGINE_CODES = {"auto": 0, "dmma": 1, "int8": 2}
ENGINE_NAMES = {1: "dmma", 2: "int8"}


def time_engine(lib, OzkProfile, code, n, d, A, B, C, sh, engine, warmup=1, steps=1):
    """One format/engine on resident inputs: (seconds per step, kernel seconds, engine)."""
    import torch
    lib.ozk_set_engine(ENGINE_CODES[engine])
    prof = OzkProfile()

    def call():
        st = lib.ozk_ozaki_gemm_device(code, n, n, n, A.data_ptr(), B.data_ptr(), d, 0.0,
                                       C.data_ptr(), sh, ctypes.byref(prof))
        if st != 0:
            raise RuntimeError(lib.ozk_last_error().decode())

    for _ in range(warmup):
        call()
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    kern = []
    e0.record(stream)
    for _ in range(steps):
        call()
        kern.append(prof.product_seconds)
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e-3 / steps, statistics.mean(kern), ENGINE_NAMES[prof.engine]


def int8_digits(fmt, l):
    """Digits per slice integer on the INT8 engine (csrc/api.cu int8_digits)."""
    if fmt != "ts":
        return 3
    return 1 if l > 1024 else 2


def engine_summary(eng, n, d, t_step, t_kern, peak_fp64, peak_i8, nd=3):
    P = d * (d + 1) // 2
    fp64_equiv = P * 2.0 * n ** 3 / t_kern / 1e12
    out = {"engine": eng, "value": round(2.0 * n ** 3 / t_step / 1e9, 3), "unit": "GFLOP/s",
           "ms_per_step": round(1e3 * t_step, 3), "slice_gemm_ms": round(1e3 * t_kern, 3),
           "slice_gemm_fp64_equiv_tflops": round(fp64_equiv, 3)}
    if eng == "dmma":
        out["slice_dgemm_frac_of_fp64_peak"] = round(fp64_equiv / peak_fp64, 4)
    else:
        i8 = nd * nd * P * 2.0 * n ** 3 / t_kern / 1e12  # nd^2 int8 digit GEMMs per pair
        out["int8_digit_gemms_per_pair"] = nd * nd
        out["int8_tensor_tops"] = round(i8, 1)
        out["frac_of_int8_peak"] = round(i8 / peak_i8, 4)
    return out


def unpin():
    """Give the main thread back every host CPU (torch's OpenMP runtime may have
    pinned it); host worker threads inherit this mask."""
    if HOST_CPUS:
        os.sched_setaffinity(0, HOST_CPUS)
    return len(HOST_CPUS) if HOST_CPUS else (os.cpu_count() or 1)


def host_inputs(lib, code, K, wdt, n, spread, pin=True):
    """gen_matrix_eq1<K>(n, n, 1) and (n, n, 2) (or the config-5 spread variant)
    from the library's host generator, into (pinned) CPU tensors."""
    import torch
    threads = unpin()
    out = []
    for seed in (1, 2):
        h = torch.empty((n, n, K), dtype=wdt, pin_memory=pin)
        st = (lib.ozk_gen_spread(code, n, n, seed, spread, h.data_ptr(), threads) if spread
              else lib.ozk_gen_eq1(code, n, n, seed, h.data_ptr(), threads))
        if st != 0:
            raise RuntimeError(lib.ozk_last_error().decode())
        out.append(h)
    return out


def cpu_leg(args, K, d, n, ha, hb, c_sub):
    """cpu_baseline of our arm: the reference CPU path on the same input bytes
    (A[:r] . B[:, :r] of this run's inputs, full-size time estimated per phase,
    see cpu_sample), its direct gemm_simple, and a bit-exact check of this run's
    GPU result C[:r, :r] against the reference's output on those bytes."""
    import numpy as np

    unpin()  # undo any pinning by torch's OpenMP runtime
    os.environ.setdefault("OMP_PROC_BIND", "close")  # read when oracle/_ref's libgomp loads
    import oracle
    cpu = oracle.best()
    cores = cpu.set_threads(len(HOST_CPUS or [1])) if hasattr(cpu, "set_threads") else 1
    r = c_sub.shape[0]
    a = np.ascontiguousarray(ha[:r].numpy())
    b = np.ascontiguousarray(hb[:, :r].numpy())
    c, wall, est, prof = cpu_sample(cpu, K, d, n, r, a, b)
    exact = bool(np.array_equal(c.view(np.uint64), c_sub.view(np.uint64)))
    if not exact:
        raise AssertionError("GPU C[:r, :r] differs from the reference ozaki_gemm on the same "
                             "inputs")
    out = {"value": round(2.0 * n ** 3 / est / 1e9, 4), "unit": "GFLOP/s", "cores": cores,
           "kind": cpu.kind,
           "sample": f"{NAMES[args.format]} Ozaki sub-GEMM A[:{r}] . B[:, :{r}] of this run's "
                     f"inputs, D={d}, one call ({wall:.2f} s: split {prof[0]:.2f} s, products "
                     f"{prof[1]:.2f} s, accumulate {prof[2]:.2f} s); full n x n time estimated "
                     f"per phase (split x n/r, products + accumulation x (n/r)^2) = {est:.1f} s",
           "host": host_cpu_info(),
           "full_size_measured": full_size_record(args.format),
           "parity": {"checked": f"GPU C[:{r}, :{r}] (this run) vs reference ozaki_gemm on "
                                 "the same bytes", "bit_exact": exact}}
    if not args.no_cpu_direct:
        out["direct"] = cpu_direct(cpu, K, n, args.cpu_direct_n, ha.numpy(), hb.numpy())
    return out


def run_ours(args):
    import torch

    rank, world, local = dist_env()
    # OZK_BENCH_ONE_DEVICE=1 is a test hook: every rank on cuda:0 with gloo
    # (NCCL refuses two ranks on one GPU), to exercise the N > 1 code path on a
    # one-GPU box; timings from it are not scaling numbers
    one_dev = os.environ.get("OZK_BENCH_ONE_DEVICE") == "1"
    torch.cuda.set_device(0 if one_dev else local)
    from paper_2301_09960_b200 import lib
    from paper_2301_09960_b200._lib import OzkProfile

    code, K, d0, wb = fmt_info(args.format)
    d = args.d or d0
    n = args.n
    P = d * (d + 1) // 2
    stream = torch.cuda.current_stream()
    wdt = torch.float32 if wb == 4 else torch.float64
    sh = stream.cuda_stream
    lib.ozk_set_engine(ENGINE_CODES[args.engine])

    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("gloo" if one_dev else "nccl")
        from paper_2301_09960_b200.sharded import ShardedOzaki
        eng = ShardedOzaki(code, n, n, n, d, rank, world)

    def check(st):
        if st != 0:
            raise RuntimeError(lib.ozk_last_error().decode())

    # the reference's inputs (gen_matrix_eq1 seeds 1, 2), generated bit-identically
    # on the host into pinned buffers (outside the timed region), then resident
    ha, hb = host_inputs(lib, code, K, wdt, n, args.spread)
    A = ha.to("cuda", non_blocking=False)
    B = hb.to("cuda", non_blocking=False)

    peak_fp64 = lib.ozk_probe_dmma_tflops(20000, sh)
    peak_i8 = lib.ozk_probe_i8_tops(4000, sh)

    if world == 1:
        C = torch.empty((n, n, K), dtype=wdt, device="cuda")

        def step(prof):
            check(lib.ozk_ozaki_gemm_device(code, n, n, n, A.data_ptr(), B.data_ptr(), d, 0.0,
                                            C.data_ptr(), sh, ctypes.byref(prof)))
    else:
        def step(prof):
            eng.run(A, B, prof)

    prof = OzkProfile()
    for _ in range(args.warmup):
        step(prof)
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    clocks = ClockSampler(0 if one_dev else local)
    clocks.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    kern, split = [], []
    e0.record(stream)
    for _ in range(args.steps):
        step(prof)
        kern.append(prof.product_seconds)
        split.append(prof.split_seconds)
    e1.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    clk = clocks.stop()
    t_step = e0.elapsed_time(e1) * 1e-3 / args.steps
    if world > 1:
        t = torch.tensor([t_step], device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        t_step = float(t.item())
    engine_used = ENGINE_NAMES.get(prof.engine, "dmma") if world == 1 else eng.engine
    value = 2.0 * n ** 3 / t_step / 1e9
    t_kern = statistics.mean(kern)
    rows_local = n if world == 1 else eng.rows_local
    fp64_work = P * 2.0 * rows_local * n * n
    nd = int8_digits(args.format, n)
    traffic = None
    traffic_src = None
    tfile = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles",
                         "r02_i8_td8192_traffic.json")
    if (engine_used == "int8" and world == 1 and args.format == "td" and n == 8192 and d == 9
            and args.spread == 0 and os.path.exists(tfile)):
        # dram__bytes_read.sum + dram__bytes_write.sum of this kernel on this
        # workload from the committed ncu --set full capture (per launch)
        tj = json.load(open(tfile))
        traffic = tj["dram_bytes_read"] + tj["dram_bytes_write"]
        traffic_src = tj["source"]
    if engine_used == "int8":
        kern_work = nd * nd * fp64_work  # nd^2 int8 digit GEMMs per slice pair
        achieved = kern_work / t_kern / 1e12
        # Denominator (B200_PROFILING.md): the driver-measured MEASURED_PEAKS.json
        # figure, sustained variant for a kernel timed inside a long step.  It has
        # bf16 only; B200 dense INT8 = 2 x dense bf16 (4.5 POPS vs 2.25 PF), so
        # the INT8 ceiling is 2 x bf16_tflops_sustained ("of measured").  The
        # in-run kind::i8 probe (no operand traffic, not power-capped: a burst
        # figure near nominal) is reported beside it.
        pk = os.path.join(os.path.dirname(os.path.abspath(__file__)), "MEASURED_PEAKS.json")
        bf16_sus = json.load(open(pk)).get("bf16_tflops_sustained") if os.path.exists(pk) else None
        peak = 2.0 * bf16_sus if bf16_sus else peak_i8
        roof = {"bound": "tensor", "kernel": "pair_gemm_i8_kernel (tcgen05.mma kind::i8 + K-word "
                "epilogue)", "achieved": round(achieved, 2),
                "peak": round(peak, 2), "unit": "TFLOP/s", "frac": round(achieved / peak, 4),
                "traffic": traffic,
                "traffic_unit": "DRAM bytes per launch", "traffic_source": traffic_src,
                "work_per_launch": f"{nd*nd}*P*2*m*n*l = {kern_work:.4g} int8 tensor ops "
                                   "(counted like flops: 2 per multiply-add)",
                "peak_source": ("of measured: 2 x MEASURED_PEAKS.json bf16_tflops_sustained = "
                                f"2 x {bf16_sus} (B200 dense INT8 = 2 x dense bf16; sustained: "
                                "the kernel runs inside back-to-back steps at the 1 kW cap)")
                if bf16_sus else "in-run kind::i8 probe (MEASURED_PEAKS.json absent)",
                "in_run_i8_probe_tops": round(peak_i8, 2),
                "frac_of_in_run_i8_probe": round(achieved / peak_i8, 4),
                "in_run_i8_probe_source": "ozk_probe_i8_tops: M=128 N=256 kind::i8 MMAs from "
                                          "resident smem, one CTA per SM, no operand traffic "
                                          "(burst, not power-capped); nominal dense INT8 4.5 POPS"}
    else:
        roof = {"bound": "tensor", "kernel": "pair_gemm_kernel (DMMA + K-word epilogue)",
                "achieved": round(fp64_work / t_kern / 1e12, 3), "peak": round(peak_fp64, 3),
                "unit": "TFLOP/s", "frac": round(fp64_work / t_kern / 1e12 / peak_fp64, 4),
                "traffic": None, "work_per_launch": f"P*2*m*n*l = {fp64_work:.4g} flop",
                "peak_source": "FP64 DMMA ceiling measured in this run (ozk_probe_dmma_tflops: "
                               "register-resident mma.m8n8k4.f64 on all SMs); MEASURED_PEAKS.json "
                               "has no FP64 figure; nominal B200 FP64 tensor 40 TF"}

    e2e = None
    if not args.no_e2e and world == 1:
        e2e = run_e2e(args, lib, OzkProfile, ha, hb, code, K, wb, d, n, C)
    elif not args.no_e2e:
        e2e = run_e2e_sharded(args, eng, A, B, K, wb, n)

    engines = {}
    variants = []
    if world == 1:
        # both slice-product engines on the same resident inputs (results are
        # bit-identical; the DMMA run carries the BASELINE metric's "slice DGEMM %
        # of FP64 peak")
        for e in ("dmma", "int8"):
            if e == engine_used:
                engines[e] = engine_summary(e, n, d, t_step, t_kern, peak_fp64, peak_i8, nd)
            elif not args.no_engine_compare:
                ts, tk, used = time_engine(lib, OzkProfile, code, n, d, A, B, C, sh, e)
                engines[e] = engine_summary(used, n, d, ts, tk, peak_fp64, peak_i8, nd)
        lib.ozk_set_engine(ENGINE_CODES[args.engine])
        r = min(args.cpu_sample, n)
        c_sub = C[:r, :r].cpu().numpy()  # for the bit-exact check against the CPU arm
        del C
        for fmt in [v for v in args.variants.split(",") if v and v != args.format]:
            variants.append(run_variant(lib, OzkProfile, fmt, n, peak_fp64, peak_i8, sh, args))

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline and args.format != "ts":
        cpu = cpu_leg(args, K, d, n, ha, hb, c_sub)

    if rank == 0:
        dm = engines.get("dmma", {})
        line = {
            "metric": METRIC, "value": round(value, 3), "unit": "GFLOP/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(1e3 * t_step, 3),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": DATA,
            "config": config_of(args, K, d, n), "engine": engine_used,
            "slice_dgemm_frac_of_fp64_peak": dm.get("slice_dgemm_frac_of_fp64_peak"),
            "phases_ms": {"split": round(1e3 * statistics.mean(split), 3),
                          "slice_gemm_fused_accumulate": round(1e3 * t_kern, 3)},
            "roofline": roof,
            "engines": engines,
            "gpu_launches": KERNELS_PER_STEP * args.steps,
            "clocks": clk,
            "e2e": e2e,
            "cpu_baseline": cpu,
            "variants": variants,
        }
        if world == 1 and args.format != "ts":
            line["direct_kword_gemm"] = direct_rate(lib, code, K, sh)
        # split (K1) against HBM: algorithmic bytes = read the K-word A and B
        # once + write the slice representation (INT8 digit planes + one int32
        # exponent per row/col and slice, or FP64 slices) -- SURVEY §8d
        rows_a = rows_local
        elems = rows_a * n + n * n if world == 1 else rows_a * n + n * (eng.plan.c1 - eng.plan.c0)
        per_elem = K * wb + (d * nd if engine_used == "int8" else d * 8)
        split_bytes = elems * per_elem + (rows_a + n) * d * 4
        t_split = statistics.mean(split)
        hbm_peak = None
        pk = os.path.join(os.path.dirname(os.path.abspath(__file__)), "MEASURED_PEAKS.json")
        if os.path.exists(pk):
            hbm_peak = json.load(open(pk)).get("hbm_gbs")
        gbs = split_bytes / t_split / 1e9 if t_split > 0 else None
        line["split_hbm"] = {
            "algorithmic_bytes": int(split_bytes), "ms": round(1e3 * t_split, 3),
            "GB/s": round(gbs, 1) if gbs else None, "peak_GB/s": hbm_peak,
            "frac": round(gbs / hbm_peak, 4) if gbs and hbm_peak else None,
            "note": "ALU-bound (K-word residual updates), not HBM-bound: profiles/r01_ncu_summary.md"}
        print(json.dumps(line), flush=True)
        if args.csv:
            from paper_2301_09960_b200.bench_csv import HEADER, BenchRecord, csv_line
            rec = BenchRecord(algo="ozaki", precision=args.format, n=n, split_count=d,
                              threads=world, seed=1, reps=args.steps,
                              t_split=statistics.mean(split), t_product=t_kern, t_accum=0.0,
                              t_total=t_step)
            new_file = not os.path.exists(args.csv)
            with open(args.csv, "a") as f:
                if new_file:
                    f.write(HEADER + "\n")
                f.write(csv_line(rec) + "\n")
    lib.ozk_set_engine(0)
    if world > 1:
        torch.distributed.destroy_process_group()
    return 0


def run_e2e(args, lib, OzkProfile, ha, hb, code, K, wb, d, n, C_dev=None):
    """Same metric through the host-buffer C-ABI entry point (ozk_ozaki_gemm):
    H2D of A and B, the GEMM, D2H of C, every step.  From pinned memory (the
    contract's e2e) and, as `pageable`, from ordinary pageable numpy buffers --
    what a drop-in caller's DenseMatrix storage is (staged through pinned slots
    inside the library, csrc/staging.cu)."""
    import numpy as np
    import torch
    hc = torch.empty((n, n, K), dtype=ha.dtype).pin_memory()
    prof = OzkProfile()

    def timed(a_ptr, b_ptr, c_ptr):
        def call():
            st = lib.ozk_ozaki_gemm(code, n, n, n, a_ptr, b_ptr, d, 0.0, c_ptr, ctypes.byref(prof))
            if st != 0:
                raise RuntimeError(lib.ozk_last_error().decode())
        call()
        times = []
        for _ in range(args.steps):
            t0 = time.perf_counter()
            call()
            times.append(time.perf_counter() - t0)
        return statistics.mean(times)

    t = timed(ha.data_ptr(), hb.data_ptr(), hc.data_ptr())
    same_dev = None
    if C_dev is not None:  # the host path's C must equal the timed device-resident C
        same_dev = bool(torch.equal(hc.to(C_dev.device).view(torch.int32),
                                    C_dev.view(torch.int32)))
        if not same_dev:
            raise AssertionError("ozk_ozaki_gemm (host buffers) differs from the device path")
    out = {"value": round(2.0 * n ** 3 / t / 1e9, 3), "unit": "GFLOP/s",
           "c_identical_to_device_run": same_dev,
           "h2d_bytes_per_step": 2 * n * n * K * wb, "d2h_bytes_per_step": n * n * K * wb,
           "ms_per_step": round(1e3 * t, 3), "api": "ozk_ozaki_gemm (host buffers, pinned)",
           "engine": ENGINE_NAMES.get(prof.engine, "?")}
    if not args.no_e2e_pageable:
        pa = np.array(ha.numpy(), copy=True)  # ordinary (pageable) heap memory
        pb = np.array(hb.numpy(), copy=True)
        pc = np.empty_like(pa)
        tp = timed(pa.ctypes.data, pb.ctypes.data, pc.ctypes.data)
        same = bool(np.array_equal(pc.view(np.uint8), hc.numpy().view(np.uint8)))
        out["pageable"] = {"value": round(2.0 * n ** 3 / tp / 1e9, 3), "unit": "GFLOP/s",
                           "ms_per_step": round(1e3 * tp, 3),
                           "vs_pinned": round(t / tp, 4),
                           "api": "ozk_ozaki_gemm (host buffers, pageable: numpy heap arrays, "
                                  "as DenseMatrix storage)",
                           "c_identical_to_pinned_run": same}
        del pa, pb, pc
    return out


def run_e2e_sharded(args, eng, A, B, K, wb, n):
    """N > 1: the same metric through the sharded public path with host
    buffers (ShardedOzaki.run_host): every step each rank brings its B column
    block and its A rows from pinned host memory, splits, all-gathers the B
    digit planes, runs its pair GEMMs and reads its C rows back, transfers
    overlapped with compute (B first, A and C in row bands); time = max over
    ranks (device events bracketing the copies)."""
    import torch
    import torch.distributed as dist
    p = eng.plan
    ha = A[p.r0:p.r1].cpu().pin_memory()
    hb = B[:, p.c0:p.c1].contiguous().cpu().pin_memory() if p.c1 > p.c0 else None
    hc = torch.empty((max(p.rows_local, 1), n, K), dtype=A.dtype).pin_memory()
    stream = torch.cuda.current_stream()

    def step():
        eng.run_host(ha, hb, hc)

    step()
    torch.cuda.synchronize()
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    t = torch.tensor([e0.elapsed_time(e1) * 1e-3 / args.steps], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    t = float(t.item())
    io = torch.tensor([(p.rows_local * n + n * (p.c1 - p.c0)) * K * wb,
                       p.rows_local * n * K * wb], dtype=torch.float64, device="cuda")
    dist.all_reduce(io)  # whole-job bytes per step (every rank's copies)
    return {"value": round(2.0 * n ** 3 / t / 1e9, 3), "unit": "GFLOP/s",
            "h2d_bytes_per_step": int(io[0].item()), "d2h_bytes_per_step": int(io[1].item()),
            "ms_per_step": round(1e3 * t, 3),
            "api": "ShardedOzaki.run_host (sharded.py), pinned host buffers, per rank; max over ranks",
            "engine": eng.engine}


def direct_rate(lib, code, K, sh, nd=1024):
    """Direct K-word GEMM comparator (gemm_simple<MultiFloat<K>> on the GPU,
    csrc/direct.cu, bit-identical to the reference's): effective GFLOP/s at nd
    (its cost is cubic; the rate carries to n = 8192, where one call would take
    minutes for QD)."""
    import torch
    ha, hb = host_inputs(lib, code, K, torch.float64, nd, 0, pin=False)
    A, B = ha.cuda(), hb.cuda()
    C = torch.empty_like(A)
    stream = torch.cuda.current_stream()

    def call():
        if lib.ozk_direct_gemm_device(code, nd, nd, nd, A.data_ptr(), B.data_ptr(), C.data_ptr(),
                                      sh) != 0:
            raise RuntimeError(lib.ozk_last_error().decode())
    call()  # warm-up
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    call()
    e1.record(stream)
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) * 1e-3
    return {"value": round(2.0 * nd ** 3 / t / 1e9, 3), "unit": "GFLOP/s", "n": nd,
            "ms": round(1e3 * t, 3),
            "kernel": "direct_gemm_kernel (gemm_simple<MultiFloat<K>>, csrc/direct.cu)"}


def run_variant(lib, OzkProfile, fmt, n, peak_fp64, peak_i8, sh, args):
    import torch
    code, K, d, wb = fmt_info(fmt)
    wdt = torch.float32 if wb == 4 else torch.float64
    ha, hb = host_inputs(lib, code, K, wdt, n, args.spread, pin=False)
    A, B = ha.cuda(), hb.cuda()
    del ha, hb
    C = torch.empty((n, n, K), dtype=wdt, device="cuda")
    out = {"workload": f"{NAMES[fmt]} Ozaki GEMM n={n} D={d}"}
    engs = ("dmma", "int8")
    for e in engs:
        ts, tk, used = time_engine(lib, OzkProfile, code, n, d, A, B, C, sh, e)
        out[e] = engine_summary(used, n, d, ts, tk, peak_fp64, peak_i8, int8_digits(fmt, n))
    lib.ozk_set_engine(ENGINE_CODES[args.engine])
    best = min((out[e] for e in engs), key=lambda r: r["ms_per_step"])
    out["value"], out["unit"], out["engine"] = best["value"], "GFLOP/s", best["engine"]
    if fmt != "ts":
        out["direct_kword_gemm"] = direct_rate(lib, code, K, sh)
    if fmt == "ts":
        # config 4 comparator: the direct triple-single GEMM kernel on the same inputs
        stream = torch.cuda.current_stream()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

        def direct():
            st = lib.ozk_ts_direct_gemm_device(n, n, n, A.data_ptr(), B.data_ptr(), C.data_ptr(),
                                               sh)
            if st != 0:
                raise RuntimeError(lib.ozk_last_error().decode())
        direct()
        e0.record(stream)
        direct()
        e1.record(stream)
        torch.cuda.synchronize()
        td = e0.elapsed_time(e1) * 1e-3
        out["direct_ts_gemm"] = {"value": round(2.0 * n ** 3 / td / 1e9, 3), "unit": "GFLOP/s",
                                 "ms_per_step": round(1e3 * td, 3),
                                 "kernel": "ts_direct_kernel (FP32 SIMT, csrc/ts_direct.cu)"}
    return out


def main():
    args = parse()
    if args.impl == "reference":
        # the reference's OpenMP loops on all host threads, bound close (SURVEY
        # §8d protocol); read by libgomp when oracle/_ref loads
        os.environ.setdefault("OMP_PROC_BIND", "close")
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
