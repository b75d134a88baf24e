"""Multi-rank C block-row sharding on CPU (gloo, world_size 2 and 3).

The sharding engine (paper_2301_09960_b200/sharded.py) runs unchanged; only
its four device operations are replaced by oracle-backed CPU equivalents
(split into the slice layout, exact slice products + the reference K-word
accumulation).  Each rank's C rows must be bit-identical to the rows of the
single-process reference ozaki_gemm -- the SURVEY §8e determinism claim --
including uneven row/column partitions and drop-threshold pruning (which
needs the all-reduce of slice maxima).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


class OracleOps:
    def __init__(self, port):
        self.port = port
        self.device = torch.device("cpu")

    def zeros(self, shape, dtype=torch.float64):
        return torch.zeros(shape, dtype=dtype)

    def split(self, K, mat, rows, cols, ld, d, side, out, pmax):
        arr = mat.contiguous().numpy().reshape(rows, cols, K)
        pieces, _ = self.port.split(K, arr, d, side)
        if side == 0:
            out[:, :rows, :cols] = torch.from_numpy(pieces)
        else:
            out[:, :cols, :rows] = torch.from_numpy(pieces.transpose(0, 2, 1).copy())
        if pmax is not None:
            mx = torch.from_numpy(np.abs(pieces).reshape(d, -1).max(axis=1))
            pmax.copy_(torch.maximum(pmax, mx))

    def gemm(self, plan, sa, sb_all, pairs, c):
        K, l, n = plan.K, plan.l, plan.n
        mr = plan.rows_local
        bt = sb_all[:, :, :, :l].permute(1, 0, 2, 3).reshape(plan.d, plan.world * plan.ncb, l)
        acc = np.zeros((mr * n, K))
        for (a, b) in pairs:
            prod = sa[a, :mr, :l].numpy() @ bt[b, :n].numpy().T  # exact on split slices
            acc = self.port.mf_add_double(K, acc, prod.reshape(-1))
        c[:mr] = torch.from_numpy(acc.reshape(mr, n, K))


class OracleDigitOps(OracleOps):
    """The INT8-engine data path of ShardedOzaki (digit-plane buffers, the
    per-plane gathers into the [D][nd][W*ncb] operand layout, plane strides) with
    the oracle's binary64 slices standing in for the digit planes (nd = 1,
    float64 "digits") -- the layout logic is shape-generic; the digit encoding
    itself is checked on the GPU (tests/test_gpu_parity.py)."""

    def int8_layout(self, K, l, d):
        return (1, l + (l & 1))

    def digit_planes(self, d, nd, rows, ld8):
        return torch.zeros((d, nd, rows, ld8), dtype=torch.float64), \
            torch.zeros((d, rows), dtype=torch.int32)

    def split_digits(self, K, mat, rows, cols, ld, d, side, digits, exps, pmax):
        self.split(K, mat, rows, cols, ld, d, side, digits[:, 0], pmax)
        exps.fill_(7)  # gathered alongside, checked in gemm_digits

    def gemm_digits(self, plan, a8, ga, b8, gb, pairs, c):
        assert b8.shape[2] == plan.world * plan.ncb and bool((gb[:, :plan.n] == 7).all())
        assert a8.shape[2] >= plan.rows_local and bool((ga == 7).all())
        K, l, n = plan.K, plan.l, plan.n
        mr = plan.rows_local
        acc = np.zeros((mr * n, K))
        for (a, b) in pairs:
            prod = a8[a, 0, :mr, :l].numpy() @ b8[b, 0, :n, :l].numpy().T
            acc = self.port.mf_add_double(K, acc, prod.reshape(-1))
        c[:mr] = torch.from_numpy(acc.reshape(mr, n, K))


    def gemm_digit_cols(self, plan, a8, ga, b8, gb, b_row0, col0, col1, pairs, c):
        """C columns [col0, col1): the local B block (b8 = this rank's planes,
        while the gather is in flight) or gathered rows [b_row0, ...)."""
        assert b8.shape[2] in (plan.ncb, plan.world * plan.ncb)
        assert b8.shape[2] == plan.world * plan.ncb or (b_row0, col0, col1) == (0, plan.c0, plan.c1)
        self.cols_done = getattr(self, "cols_done", []) + [(col0, col1)]
        K, l, w = plan.K, plan.l, col1 - col0
        mr = plan.rows_local
        acc = np.zeros((mr * w, K))
        for (a, b) in pairs:
            prod = a8[a, 0, :mr, :l].numpy() @ b8[b, 0, b_row0:b_row0 + w, :l].numpy().T
            acc = self.port.mf_add_double(K, acc, prod.reshape(-1))
        c[:mr, col0:col1] = torch.from_numpy(acc.reshape(mr, w, K))


def _worker(rank, world, port_num, cases, q, digits=False):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port_num)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        from paper_2301_09960_b200.sharded import ShardedOzaki
        port = oracle.load_port()
        for (K, m, l, n, d, drop) in cases:
            a = port.gen_eq1(K, m, l, 31 + m)
            b = port.gen_eq1(K, l, n, 32 + m)
            want = port.ozaki_gemm(K, a, b, d, drop)
            ops = OracleDigitOps(port) if digits else OracleOps(port)
            eng = ShardedOzaki(K, m, l, n, d, rank, world, ops=ops, drop_threshold=drop)
            assert eng.engine == ("int8" if digits else "dmma")
            got = eng.run(torch.from_numpy(a), torch.from_numpy(b)).numpy()
            r0, r1 = eng.plan.r0, eng.plan.r1
            ok = np.array_equal(got.view(np.uint64), want[r0:r1].view(np.uint64))
            if digits and r1 > r0 and eng.plan.c1 > eng.plan.c0:
                # the local block went first, then the rest: every column once
                cols = sorted(ops.cols_done)
                ok = ok and cols[0][0] == 0 and cols[-1][1] == n and all(
                    x[1] == y[0] for x, y in zip(cols, cols[1:]))
            q.put((rank, (K, m, l, n, d, drop), bool(ok)))
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("digits", [False, True], ids=["fp64-slices", "digit-planes"])
@pytest.mark.parametrize("world", [2, 3, 8])
def test_sharded_matches_single_process(world, digits):
    cases = [(2, 10, 12, 9, 4, 0.0), (3, 7, 9, 11, 5, 0.0), (2, 13, 16, 14, 5, 2.0 ** -60),
             (4, 5, 6, 4, 6, 0.0)]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    mp.spawn(_worker, args=(world, _free_port(), cases, q, digits), nprocs=world, join=True)
    results = [q.get() for _ in range(world * len(cases))]
    bad = [r for r in results if not r[2]]
    assert not bad, bad


def test_block_range_partition():
    from paper_2301_09960_b200.sharded import ShardPlan, block_range
    for total in (1, 7, 8, 8192, 8193):
        for parts in (1, 2, 3, 8):
            spans = [block_range(total, parts, i) for i in range(parts)]
            assert spans[0][0] == 0 and spans[-1][1] == total
            assert all(spans[i][1] == spans[i + 1][0] for i in range(parts - 1))
            assert max(b - a for a, b in spans) - min(b - a for a, b in spans) <= 1
    p = ShardPlan(2, 10, 7, 9, 3, 2, 3)
    assert p.ncb == 3 and (p.c0, p.c1) == (6, 9) and p.ld == 8
