"""C block-row sharding of one Ozaki GEMM across the GPUs of a node.

Rank r of W owns C rows [r0, r1) and B columns [c0, c1):

1. split its A row block on its own GPU (per-row split: bit-identical to the
   rows of the global split, ozaki.hpp:102-103);
2. split its B column block (per-column split: bit-identical to the columns of
   the global split);
3. all-gather the B slices over NCCL (NVLink/NVSwitch) -- the path's one real
   exchange step: D * l * ceil(n/W) * 8 bytes per rank (INT8 digits: D * nd *
   l * ceil(n/W)); B is split first and the gather runs on a side stream while
   the A rows are split;
4. with drop_threshold > 0, all-reduce(max) the per-slice maxima so every rank
   prunes the same pairs (ozaki.hpp:198-221);
5. run every slice pair for its rows with the fused accumulation -- with the
   INT8 engine first for its own B column block while the all-gather is still
   in flight, then for the gathered columns.  The per-element accumulation
   order is unchanged, so C is bit-identical for any number of GPUs.

Two slice representations, bit-identical results:
* INT8 engine (default where it applies, ozk_int8_digits > 0): the splits write
  nd int8 digit planes + one grid exponent per row/column
  (ozk_split_digits_device_async), the all-gather moves D*nd*l*ceil(n/W)
  bytes per rank (2.7x less than FP64 slices), one collective per digit plane
  straight into the [D][nd][W*ncb][ld8] operand layout (each plane's rank
  blocks are contiguous rows, so no re-layout copy), and
  ozk_digits_gemm_device_async runs the pairs on tcgen05.  Nothing in the
  device path synchronises the stream; the split's data-error flags are
  checked once at the end of run();
* DMMA engine: FP64 slices (ozk_split_slices_device / ozk_slices_gemm_device).

The gathered B slices stay in the layout the all-gather produces
([W][D][ncb][ld]); the GEMM kernel addresses column j in block j // ncb
directly (ozk_slices_gemm_device), so no re-layout copy is needed.

Device work goes through an ``ops`` object; :class:`GpuOps` drives libozk.so.
The CPU tests substitute an oracle-backed implementation of the same four
operations to check the partitioning, padding, gather layout and pair logic
with the gloo backend.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import torch
import torch.distributed as dist


def block_range(total: int, parts: int, idx: int) -> tuple[int, int]:
    """Contiguous near-equal partition (first total % parts blocks get one more)."""
    base, extra = divmod(total, parts)
    lo = idx * base + min(idx, extra)
    return lo, lo + base + (1 if idx < extra else 0)


def triangular_pairs(d: int) -> list[tuple[int, int]]:
    return [(a, b) for a in range(d) for b in range(d - a)]


def pruned_pairs(d, amax, bmax, drop) -> list[tuple[int, int]]:
    """ozaki.hpp:198-221."""
    lead = amax[0] * bmax[0]
    out = []
    for a in range(d):
        for b in range(d - a):
            if drop > 0.0 and amax[a] * bmax[b] < drop * lead:
                continue
            out.append((a, b))
    return out


OZK_TS = 0x103


@dataclass
class ShardPlan:
    K: int          # ozk_format code: 2/3/4 (DD/TD/QD) or 0x103 (TS)
    m: int
    l: int
    n: int
    d: int
    rank: int
    world: int

    def __post_init__(self):
        self.r0, self.r1 = block_range(self.m, self.world, self.rank)
        self.ncb = -(-self.n // self.world)          # columns per B block (padded)
        self.c0 = min(self.rank * self.ncb, self.n)
        self.c1 = min(self.c0 + self.ncb, self.n)
        self.ld = (self.l + 1) & ~1                  # ozk_slice_ld

    @property
    def rows_local(self) -> int:
        return self.r1 - self.r0

    @property
    def words(self) -> int:
        return 3 if self.K == OZK_TS else self.K


class GpuOps:
    """libozk.so device entry points on torch CUDA tensors (current stream)."""

    def __init__(self):
        from ._lib import lib
        self.lib = lib
        self.device = torch.device("cuda", torch.cuda.current_device())
        # split data-error flags (A rows, B columns) of the asynchronous entries
        self.flags = torch.zeros(2, dtype=torch.int32, device=self.device)

    def reset_flags(self):
        self.flags.zero_()

    def check_flags(self):
        """Non-finite / too-large entries found by the splits (A first, as
        split_matrix(a) runs before split_matrix(b)); synchronises the stream."""
        for i in (0, 1):
            self._check(self.lib.ozk_check_split_flag(self.flags.data_ptr() + 4 * i,
                                                      self._stream()))

    def _check(self, st):
        if st != 0:
            raise RuntimeError(self.lib.ozk_last_error().decode())

    def _stream(self):
        return torch.cuda.current_stream().cuda_stream

    def zeros(self, shape, dtype=torch.float64):
        return torch.zeros(shape, dtype=dtype, device=self.device)

    def split(self, K, mat, rows, cols, ld, d, side, out, pmax):
        """mat: tensor view whose data_ptr is element (0,0); row stride ld elements.
        out: (d, plane_rows, ld_slice) slices; plane_rows may exceed the outer dim."""
        self._check(self.lib.ozk_split_slices_device(
            K, rows, cols, ld, mat.data_ptr(), d, side, out.data_ptr(), out.shape[1],
            pmax.data_ptr() if pmax is not None else None, self._stream()))

    def gemm(self, plan: ShardPlan, sa, sb_all, pairs, c):
        flat = (ctypes.c_int * (2 * len(pairs)))(*[v for p in pairs for v in p])
        self._check(self.lib.ozk_slices_gemm_device(
            plan.K, plan.rows_local, plan.l, plan.n, sa.data_ptr(), sb_all.data_ptr(), plan.ncb,
            plan.world, plan.d * plan.ncb * plan.ld, plan.d, flat, len(pairs), c.data_ptr(),
            plan.n, self._stream()))

    # ---- INT8 engine ----
    def int8_layout(self, K, l, d):
        """(nd, ld8) of the digit planes, or None where the engine does not apply
        (or the DMMA engine is forced with ozk_set_engine)."""
        if self.lib.ozk_get_engine() == 1:
            return None
        nd = self.lib.ozk_int8_digits(K, l, d)
        return (nd, (l + 15) & ~15) if nd > 0 else None

    def digit_planes(self, d, nd, rows, ld8):
        return (torch.zeros((d, nd, rows, ld8), dtype=torch.int8, device=self.device),
                torch.zeros((d, rows), dtype=torch.int32, device=self.device))

    def split_digits(self, K, mat, rows, cols, ld, d, side, digits, exps, pmax):
        self._check(self.lib.ozk_split_digits_device_async(
            K, rows, cols, ld, mat.data_ptr(), d, side, digits.data_ptr(), digits.shape[3],
            digits.shape[2], exps.data_ptr(), pmax.data_ptr() if pmax is not None else None,
            self.flags.data_ptr() + 4 * side, self._stream()))

    def split_digit_rows(self, K, mat, rows, cols, ld, d, side, digits, r0, exps):
        """split_digits into rows [r0, r0 + rows) of full-height digit planes."""
        ld8, plane_rows = digits.shape[3], digits.shape[2]
        self._check(self.lib.ozk_split_digits_device_async(
            K, rows, cols, ld, mat.data_ptr(), d, side, digits.data_ptr() + r0 * ld8, ld8,
            plane_rows, exps.data_ptr() + 4 * r0, None, self.flags.data_ptr() + 4 * side,
            self._stream()))

    def gemm_digit_block(self, plan: ShardPlan, r0, rows, a8, ga, b8, gb, b_row0, col0, col1,
                         pairs, c):
        """C rows [r0, r0 + rows) x columns [col0, col1), B digits from plane rows
        [b_row0, ...) of b8."""
        flat = (ctypes.c_int * (2 * len(pairs)))(*[v for p in pairs for v in p])
        ld8, esz = a8.shape[3], c.element_size() * c.shape[2]
        self._check(self.lib.ozk_digits_gemm_device_async(
            plan.K, rows, plan.l, col1 - col0, a8.data_ptr() + r0 * ld8, ga.data_ptr() + 4 * r0,
            a8.shape[2], b8.data_ptr() + b_row0 * ld8, gb.data_ptr() + 4 * b_row0, b8.shape[2],
            ld8, plan.d, flat, len(pairs), c.data_ptr() + (r0 * plan.n + col0) * esz, plan.n,
            self._stream()))

    def gemm_digit_rows(self, plan: ShardPlan, r0, rows, a8, ga, b8, gb, pairs, c):
        """gemm_digits for C rows [r0, r0 + rows) of this rank (c: all its rows)."""
        flat = (ctypes.c_int * (2 * len(pairs)))(*[v for p in pairs for v in p])
        ld8, esz = a8.shape[3], c.element_size() * c.shape[2]
        self._check(self.lib.ozk_digits_gemm_device_async(
            plan.K, rows, plan.l, plan.n, a8.data_ptr() + r0 * ld8, ga.data_ptr() + 4 * r0,
            a8.shape[2], b8.data_ptr(), gb.data_ptr(), b8.shape[2], ld8, plan.d, flat, len(pairs),
            c.data_ptr() + r0 * plan.n * esz, plan.n, self._stream()))

    def gemm_digit_cols(self, plan: ShardPlan, a8, ga, b8, gb, b_row0, col0, col1, pairs, c):
        """gemm_digits for C columns [col0, col1) of this rank's rows, B digits from
        plane rows [b_row0, b_row0 + col1 - col0) of b8 (its own plane height)."""
        self.gemm_digit_block(plan, 0, plan.rows_local, a8, ga, b8, gb, b_row0, col0, col1,
                              pairs, c)

    def gemm_digits(self, plan: ShardPlan, a8, ga, b8, gb, pairs, c):
        flat = (ctypes.c_int * (2 * len(pairs)))(*[v for p in pairs for v in p])
        self._check(self.lib.ozk_digits_gemm_device_async(
            plan.K, plan.rows_local, plan.l, plan.n, a8.data_ptr(), ga.data_ptr(), a8.shape[2],
            b8.data_ptr(), gb.data_ptr(), b8.shape[2], a8.shape[3], plan.d, flat, len(pairs),
            c.data_ptr(), plan.n, self._stream()))


class ShardedOzaki:
    """One rank's part of a C block-row sharded Ozaki GEMM."""

    def __init__(self, K, m, l, n, d, rank, world, ops=None, group=None, drop_threshold=0.0):
        self.plan = ShardPlan(K, m, l, n, d, rank, world)
        self.ops = ops if ops is not None else GpuOps()
        self.group = group
        self.drop = float(drop_threshold)
        p = self.plan
        layout = self.ops.int8_layout(K, l, d) if hasattr(self.ops, "int8_layout") else None
        self.engine = "int8" if layout else "dmma"
        if layout:
            nd, ld8 = layout
            self.a8, self.ga = self.ops.digit_planes(d, nd, max(p.rows_local, 1), ld8)
            self.b8, self.gb = self.ops.digit_planes(d, nd, p.ncb, ld8)
            # the GEMM operand layout [D][nd][W*ncb][ld8] / [D][W*ncb], filled
            # by one all-gather per plane (rank r's block = rows r*ncb..)
            self.b8_cat, self.gb_cat = self.ops.digit_planes(d, nd, world * p.ncb, ld8)
        else:
            self.sa = self.ops.zeros((d, max(p.rows_local, 1), p.ld))
            self.sb = self.ops.zeros((d, p.ncb, p.ld))
            self.sb_all = self.ops.zeros((world, d, p.ncb, p.ld))
        self.c = self.ops.zeros((max(p.rows_local, 1), n, p.words),
                                dtype=torch.float32 if K == OZK_TS else torch.float64)
        self.pmax = self.ops.zeros((2, d)) if self.drop > 0.0 else None
        self.timing = hasattr(self.ops, "device") and self.ops.device.type == "cuda"
        self._comm = None  # side stream of the B all-gather (NCCL)

    @property
    def rows_local(self) -> int:
        return self.plan.rows_local

    def _gather(self, out, local):
        """out: world blocks of local's shape, back to back (dim 0 of out is
        world * local.shape[0] rows, or world when out has one more dim)."""
        if dist.get_backend(self.group) == "nccl":
            dist.all_gather_into_tensor(out, local, group=self.group)
        else:
            parts = list(out.reshape(self.plan.world, *local.shape).unbind(0))
            dist.all_gather(parts, local, group=self.group)

    def _all_gather(self):
        if self.engine == "int8":
            # one collective per digit plane and per exponent row: column j of
            # the gathered B is row j of every plane (the ceil partition puts
            # rank r's columns at r*ncb), so the planes land in the GEMM's
            # operand layout with no re-layout copy.  The D*nd + D calls are
            # coalesced into one NCCL group where torch offers it.
            d, nd = self.b8.shape[0], self.b8.shape[1]

            def planes():
                for s in range(d):
                    for t in range(nd):
                        self._gather(self.b8_cat[s, t], self.b8[s, t])
                    self._gather(self.gb_cat[s], self.gb[s])

            # (torch's fast path: a block of only all_gather_into_tensor calls
            # becomes one allgather_into_tensor_coalesced = one NCCL group)
            cm = getattr(dist, "_coalescing_manager", None)
            if cm is not None and dist.get_backend(self.group) == "nccl":
                with cm(group=self.group):
                    planes()
            else:
                planes()
        else:
            self._gather(self.sb_all, self.sb)

    def run_host(self, hA, hB, hC, bands=4):
        """The same C rows from pinned HOST buffers, transfers overlapped:
        hA this rank's A rows (rows_local, l, K), hB its B column block
        (l, c1 - c0, K) contiguous, hC receives its C rows (rows_local, n, K).
        B's block crosses PCIe first on a copy stream and is split, its NCCL
        all-gather runs on a side stream while A arrives in `bands` row bands,
        each split right before its slice-GEMM band, and each band's C rows go
        back on a second copy stream while later bands compute (rows are
        independent: bit-identical to run()).  Other engines / pruning: the
        copies around run()."""
        p, ops = self.plan, self.ops
        cur = torch.cuda.current_stream()
        if self.engine != "int8" or self.pmax is not None or not p.rows_local:
            da = hA.to(self.ops.device, non_blocking=True)
            db = torch.zeros((p.l, p.n, p.words), dtype=hA.dtype, device=self.ops.device)
            if p.c1 > p.c0:
                db[:, p.c0:p.c1].copy_(hB, non_blocking=True)
            c = self.run(da, db)
            hC[: p.rows_local].copy_(c, non_blocking=True)
            return
        if getattr(self, "_host", None) is None:
            dev = self.ops.device
            self._host = dict(
                xs=torch.cuda.Stream(dev), ys=torch.cuda.Stream(dev),
                da=torch.empty((p.rows_local, p.l, p.words), dtype=hA.dtype, device=dev),
                db=torch.empty((p.l, max(p.c1 - p.c0, 1), p.words), dtype=hA.dtype, device=dev))
        h = self._host
        xs, ys, da, db = h["xs"], h["ys"], h["da"], h["db"]
        ops.reset_flags()
        nb = max(1, min(bands, p.rows_local // 256))
        bounds = [p.rows_local * q // nb for q in range(nb + 1)]
        xs.wait_stream(cur)
        ys.wait_stream(cur)
        ev_b = torch.cuda.Event()
        ev_a = [torch.cuda.Event() for _ in range(nb)]
        with torch.cuda.stream(xs):
            if p.c1 > p.c0:
                db[:, : p.c1 - p.c0].copy_(hB, non_blocking=True)
            ev_b.record(xs)
            for q in range(nb):
                da[bounds[q]:bounds[q + 1]].copy_(hA[bounds[q]:bounds[q + 1]], non_blocking=True)
                ev_a[q].record(xs)
        cur.wait_event(ev_b)
        if p.c1 > p.c0:
            ops.split_digit_rows(p.K, db, p.l, p.c1 - p.c0, p.c1 - p.c0, p.d, 1, self.b8, 0,
                                 self.gb)
        comm = None
        if dist.get_backend(self.group) == "nccl":
            if self._comm is None:
                self._comm = torch.cuda.Stream()
            comm = self._comm
            comm.wait_stream(cur)
            with torch.cuda.stream(comm):
                self._all_gather()
        else:
            self._all_gather()
        pairs = triangular_pairs(p.d)
        for q in range(nb):
            r0, r1 = bounds[q], bounds[q + 1]
            cur.wait_event(ev_a[q])
            ops.split_digit_rows(p.K, da[r0:r1], r1 - r0, p.l, p.l, p.d, 0, self.a8, r0, self.ga)
            if q == 0 and p.world > 1:
                # band 0: the local B block while the gather is in flight
                if p.c1 > p.c0:
                    ops.gemm_digit_block(p, r0, r1 - r0, self.a8, self.ga, self.b8, self.gb, 0,
                                         p.c0, p.c1, pairs, self.c)
                if comm is not None:
                    cur.wait_stream(comm)
                for lo, hi in ((0, p.c0), (p.c1, p.n)):
                    if hi > lo:
                        ops.gemm_digit_block(p, r0, r1 - r0, self.a8, self.ga, self.b8_cat,
                                             self.gb_cat, lo, lo, hi, pairs, self.c)
            else:
                if q == 0 and comm is not None:
                    cur.wait_stream(comm)
                ops.gemm_digit_rows(p, r0, r1 - r0, self.a8, self.ga, self.b8_cat, self.gb_cat,
                                    pairs, self.c)
            done = torch.cuda.Event()
            done.record(cur)
            ys.wait_event(done)
            with torch.cuda.stream(ys):
                hC[r0:r1].copy_(self.c[r0:r1], non_blocking=True)
        cur.wait_stream(ys)
        cur.wait_stream(xs)
        ops.check_flags()

    def run(self, A, B, prof=None):
        """A: (m, l, K) or this rank's rows; B: (l, n, K) full (row stride n).
        Returns this rank's C rows (rows_local, n, K)."""
        p, ops = self.plan, self.ops
        if self.timing:
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
            ev[0].record()
        a_rows = A[p.r0:p.r1] if A.shape[0] == p.m else A
        if hasattr(ops, "reset_flags"):
            ops.reset_flags()
        if self.pmax is not None:
            self.pmax.zero_()
        amax = self.pmax[0] if self.pmax is not None else None
        bmax = self.pmax[1] if self.pmax is not None else None
        # B first: its all-gather (the path's one exchange) then runs on a side
        # stream while this rank splits its A rows (NCCL; gloo gathers on the
        # host and cannot overlap)
        if p.c1 > p.c0:
            # column block [c0, c1) of the row-major (l x n) B, split in place
            if self.engine == "int8":
                ops.split_digits(p.K, B[:, p.c0:p.c1], p.l, p.c1 - p.c0, p.n, p.d, 1, self.b8,
                                 self.gb, bmax)
            else:
                ops.split(p.K, B[:, p.c0:p.c1], p.l, p.c1 - p.c0, p.n, p.d, 1, self.sb, bmax)
        comm = None
        if self.timing and dist.get_backend(self.group) == "nccl":
            if self._comm is None:
                self._comm = torch.cuda.Stream()
            comm = self._comm
            comm.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(comm):
                self._all_gather()
        else:
            self._all_gather()
        if p.rows_local:
            if self.engine == "int8":
                ops.split_digits(p.K, a_rows, p.rows_local, p.l, p.l, p.d, 0, self.a8, self.ga,
                                 amax)
            else:
                ops.split(p.K, a_rows, p.rows_local, p.l, p.l, p.d, 0, self.sa, amax)
        if self.timing:
            ev[1].record()
        if self.pmax is not None:
            if hasattr(ops, "check_flags"):
                ops.check_flags()  # the maxima are only meaningful for finite inputs
            dist.all_reduce(self.pmax, op=dist.ReduceOp.MAX, group=self.group)
            mx = self.pmax.cpu().tolist()
            pairs = pruned_pairs(p.d, mx[0], mx[1], self.drop)
        else:
            pairs = triangular_pairs(p.d)
        # INT8 engine, W > 1: this rank's own B column block is multiplied
        # while the all-gather is still in flight, the other columns after it
        # (C elements are independent: the same bits as one GEMM)
        local_first = (self.engine == "int8" and p.world > 1 and p.rows_local and pairs
                       and p.c1 > p.c0 and hasattr(ops, "gemm_digit_cols"))
        if local_first:
            ops.gemm_digit_cols(p, self.a8, self.ga, self.b8, self.gb, 0, p.c0, p.c1, pairs,
                                self.c)
        if self.timing:
            ev[4].record()
        if comm is not None:
            torch.cuda.current_stream().wait_stream(comm)
        if self.timing:
            ev[2].record()
        if p.rows_local:
            if not pairs:
                self.c.zero_()
            elif local_first:
                for lo, hi in ((0, p.c0), (p.c1, p.n)):
                    if hi > lo:
                        ops.gemm_digit_cols(p, self.a8, self.ga, self.b8_cat, self.gb_cat, lo,
                                            lo, hi, pairs, self.c)
            elif self.engine == "int8":
                ops.gemm_digits(p, self.a8, self.ga, self.b8_cat, self.gb_cat, pairs, self.c)
            else:
                ops.gemm(p, self.sa, self.sb_all, pairs, self.c)
        if hasattr(ops, "check_flags"):
            ops.check_flags()  # synchronises the stream
        if self.timing:
            ev[3].record()
            torch.cuda.current_stream().synchronize()
            if prof is not None:
                # split = both splits; transfer = the part of the all-gather
                # (+ maxima all-reduce) not hidden behind the A split and the
                # local-block GEMM; product = the GEMM work on either side
                prof.split_seconds = ev[0].elapsed_time(ev[1]) * 1e-3
                prof.transfer_seconds = ev[4].elapsed_time(ev[2]) * 1e-3
                prof.product_seconds = (ev[1].elapsed_time(ev[4]) +
                                        ev[2].elapsed_time(ev[3])) * 1e-3
                prof.accumulate_seconds = 0.0
                prof.total_seconds = ev[0].elapsed_time(ev[3]) * 1e-3
                prof.split_count = p.d
                prof.pairs = len(pairs)
                prof.gpus = p.world
                prof.engine = 2 if self.engine == "int8" else 1
        return self.c[: p.rows_local]
