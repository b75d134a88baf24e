"""The sharded path with real device ops: W = 2, 3 ranks as separate processes
on cuda:0 (gloo backend, which all-gathers CUDA tensors through the host;
NCCL refuses two ranks on one device).  Each rank runs ShardedOzaki with
GpuOps -- its splits into INT8 digit planes (or FP64 slices for l <= 128), the
gathered-plane permute and its pair GEMMs on the B200 -- and its C rows must
equal the reference's rows bit for bit, both from device tensors (run) and
from pinned host buffers with overlapped, banded transfers (run_host).  The kernels of different ranks never
wait on each other (the only exchange is the host-side collective), so sharing
one GPU changes timing, not results.
"""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _worker(rank, world, port, cases, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        import oracle
        from paper_2301_09960_b200.sharded import ShardedOzaki
        cpu = oracle.best()
        for (K, m, l, n, d, drop) in cases:
            a = cpu.gen_eq1(K, m, l, 71 + m)
            b = cpu.gen_eq1(K, l, n, 72 + m)
            want = cpu.ozaki_gemm(K, a, b, d, drop)
            eng = ShardedOzaki(K, m, l, n, d, rank, world, drop_threshold=drop)
            got = eng.run(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda())
            got = got.cpu().numpy()
            r0, r1 = eng.plan.r0, eng.plan.r1
            ok = np.array_equal(got.view(np.uint64), want[r0:r1].view(np.uint64))
            # host-buffer path (overlapped copies, A/C in row bands)
            ok_host = _host_rows_equal(eng, a, b, want)
            q.put((rank, (K, m, l, n, d, drop), eng.engine, bool(ok and ok_host)))
    finally:
        dist.destroy_process_group()


def _host_rows_equal(eng, a, b, want):
    import torch
    p = eng.plan
    ha = torch.from_numpy(a[p.r0:p.r1].copy()).pin_memory()
    hb = torch.from_numpy(b[:, p.c0:p.c1].copy()).pin_memory() if p.c1 > p.c0 else None
    hc = torch.full((max(p.rows_local, 1), p.n, p.words), float("nan"),
                    dtype=ha.dtype).pin_memory()
    for _ in range(2):  # the second call reuses the streams and buffers
        eng.run_host(ha, hb, hc, bands=3)
        torch.cuda.synchronize()
    got = hc[: p.rows_local].numpy()
    return np.array_equal(got.view(np.uint64), want[p.r0:p.r1].view(np.uint64))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_ranks_on_device(ozk, world):
    cases = [(2, 100, 600, 90, 6, 0.0), (3, 64, 1030, 70, 9, 0.0), (4, 40, 300, 50, 12, 0.0),
             (2, 70, 700, 64, 10, 2.0 ** -70), (2, 30, 100, 40, 6, 0.0),
             (3, 1600, 300, 200, 4, 0.0)]  # >= 256 rows per rank: banded host path
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    mp.spawn(_worker, args=(world, _free_port(), cases, q), nprocs=world, join=True)
    results = [q.get() for _ in range(world * len(cases))]
    bad = [r for r in results if not r[3]]
    assert not bad, bad
    engines = {r[1][2]: r[2] for r in results}
    assert engines[600] == "int8" and engines[100] == "dmma"  # keyed by l


def _nccl_single(rank, port, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1)
    try:
        import oracle
        from paper_2301_09960_b200.sharded import ShardedOzaki
        from paper_2301_09960_b200._lib import OzkProfile
        cpu = oracle.best()
        for (K, m, l, n, d, drop) in [(3, 64, 1030, 70, 9, 0.0), (2, 80, 600, 64, 8, 2.0 ** -80)]:
            a = cpu.gen_eq1(K, m, l, 81 + m)
            b = cpu.gen_eq1(K, l, n, 82 + m)
            want = cpu.ozaki_gemm(K, a, b, d, drop)
            eng = ShardedOzaki(K, m, l, n, d, 0, 1, drop_threshold=drop)
            prof = OzkProfile()
            for _ in range(2):  # the second run reuses the side stream and buffers
                got = eng.run(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda(), prof)
            ok = np.array_equal(got.cpu().numpy().view(np.uint64), want.view(np.uint64))
            ok = ok and _host_rows_equal(eng, a, b, want)
            q.put((K, eng.engine, eng._comm is not None, bool(ok), prof.engine))
    finally:
        dist.destroy_process_group()


def test_sharded_nccl_side_stream_gather(ozk):
    """The NCCL branch of ShardedOzaki.run (B all-gather + plane permute on a
    side stream overlapping the A split), on a one-rank NCCL group."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    mp.spawn(_nccl_single, args=(_free_port(), q), nprocs=1, join=True)
    res = [q.get() for _ in range(2)]
    assert all(r[3] for r in res), res
    assert all(r[2] for r in res), res  # the side stream was used
    assert all(r[1] == "int8" and r[4] == 2 for r in res), res


def _random_cases(seed, count):
    rng = np.random.default_rng(21000 + seed)
    cases = []
    for _ in range(count):
        K = int(rng.integers(2, 5))
        m = int(rng.integers(1, 900))
        n = int(rng.integers(1, 300))
        l = int(rng.integers(1, 129)) if rng.random() < 0.3 else int(rng.integers(129, 900))
        d = int(rng.integers(2, {2: 8, 3: 11, 4: 14}[K] + 1))
        drop = 0.0 if rng.random() < 0.7 else float(2.0 ** -int(rng.integers(20, 140)))
        cases.append((K, m, l, n, d, drop))
    return cases


_span_sh = os.environ.get("OZK_FUZZ_SHARD_SEEDS")
SHARD_SEEDS = list(range(*map(int, _span_sh.split(":")))) if _span_sh else [0]


@pytest.mark.parametrize("seed", SHARD_SEEDS)
@pytest.mark.parametrize("world", [2, 4])
def test_sharded_random_on_device(ozk, world, seed):
    """Seeded shapes through the sharded path on one device (gloo): ragged and
    empty row / column blocks, both engines, pruning, the local-block-first
    GEMM order, device and banded host paths -- every rank's C rows
    bit-identical to the reference."""
    cases = _random_cases(seed * 10 + world, 6)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    mp.spawn(_worker, args=(world, _free_port(), cases, q), nprocs=world, join=True)
    results = [q.get() for _ in range(world * len(cases))]
    bad = [r for r in results if not r[3]]
    assert not bad, bad
