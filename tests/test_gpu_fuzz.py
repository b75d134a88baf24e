"""Seeded randomised parity sweep of the public GEMM path against the CPU
oracle (the compiled reference where present): format DD/TD/QD/TS, ragged
shapes on both sides of the INT8 engine's l > 128 boundary, split count,
pruning threshold, Eq. (1) or exponent-spread inputs, zero rows/columns, host
or device API, auto or forced-DMMA engine.  Every C must be bit-identical to
the reference's (D >= 2; D = 1 products round, as in the reference).
"""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TS = 0x103
# $OZK_FUZZ_SEEDS=a:b runs seeds [a, b) instead (extended sweeps,
# profiles/r02_fuzz_extended.log)
_span = os.environ.get("OZK_FUZZ_SEEDS")
SEEDS = list(range(*map(int, _span.split(":")))) if _span else list(range(160))


def _case(seed):
    rng = np.random.default_rng(1000 + seed)
    fmt = [2, 3, 4, TS][seed % 4]
    m, n = (int(x) for x in rng.integers(1, 161, 2))
    l = int(rng.integers(1, 129)) if rng.random() < 0.35 else int(rng.integers(129, 701))
    dmax = {2: 8, 3: 11, 4: 14, TS: 16}[fmt]
    d = int(rng.integers(2, dmax + 1))
    drop = 0.0 if rng.random() < 0.6 else float(2.0 ** -int(rng.integers(10, 150)))
    spread = int(rng.integers(8, 200)) if (fmt != TS and rng.random() < 0.3) else 0
    zero_a = int(rng.integers(0, m)) if rng.random() < 0.25 else None
    zero_b = int(rng.integers(0, n)) if rng.random() < 0.25 else None
    device = bool(rng.random() < 0.5)
    dmma = bool(rng.random() < 0.2)
    return fmt, m, l, n, d, drop, spread, zero_a, zero_b, device, dmma


def _inputs(cpu, port, fmt, m, l, n, spread, seed):
    if fmt == TS:
        return port.gen_eq1_ts(m, l, 2 * seed + 1), port.gen_eq1_ts(l, n, 2 * seed + 2)
    if spread:
        return (port.gen_spread(fmt, m, l, 2 * seed + 1, spread),
                port.gen_spread(fmt, l, n, 2 * seed + 2, spread))
    return cpu.gen_eq1(fmt, m, l, 2 * seed + 1), cpu.gen_eq1(fmt, l, n, 2 * seed + 2)


@pytest.mark.parametrize("seed", SEEDS)
def test_random_gemm_bitexact(ozk, cpu, port, seed):
    import torch
    fmt, m, l, n, d, drop, spread, zero_a, zero_b, device, dmma = _case(seed)
    a, b = _inputs(cpu, port, fmt, m, l, n, spread, seed)
    if zero_a is not None:
        a[zero_a] = 0.0
    if zero_b is not None:
        b[:, zero_b] = 0.0
    if fmt == TS:
        want = port.ozaki_gemm_ts(a, b, d, drop)
    else:
        want = cpu.ozaki_gemm(fmt, a, b, d, drop)
    ozk.set_engine("dmma" if dmma else "auto")
    try:
        if device:
            got, _ = ozk.ozaki_gemm(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda(), d,
                                    drop_threshold=drop)
            got = got.cpu().numpy()
        else:
            got, _ = ozk.ozaki_gemm(a, b, d, drop_threshold=drop)
    finally:
        ozk.set_engine("auto")
    u = np.uint32 if fmt == TS else np.uint64
    bad = np.flatnonzero((got.view(u) != want.view(u)).reshape(m * n, -1).any(axis=1))
    assert bad.size == 0, (f"case {_case(seed)}: {bad.size} of {m * n} elements differ, "
                           f"first {divmod(int(bad[0]), n)}")


_span_mt = os.environ.get("OZK_FUZZ_MT_SEEDS")
MT_SEEDS = list(range(*map(int, _span_mt.split(":")))) if _span_mt else list(range(16))


@pytest.mark.parametrize("seed", MT_SEEDS)
def test_random_gemm_bitexact_multi_tile(ozk, cpu, port, seed):
    """Larger seeded cases (300-700 rows/columns: several tiles, waves and
    paced clusters of the INT8 engine; D <= 6 keeps the CPU oracle fast)."""
    rng = np.random.default_rng(5000 + seed)
    fmt = [2, 3, 4, TS][seed % 4]
    m, n = (int(x) for x in rng.integers(300, 701, 2))
    l = int(rng.integers(129, 1025))
    d = int(rng.integers(2, 7))
    drop = 0.0 if seed % 3 else float(2.0 ** -int(rng.integers(30, 120)))
    a, b = _inputs(cpu, port, fmt, m, l, n, 0 if seed % 5 else 60, seed + 777)
    want = (port.ozaki_gemm_ts(a, b, d, drop) if fmt == TS else cpu.ozaki_gemm(fmt, a, b, d, drop))
    got, _ = ozk.ozaki_gemm(a, b, d, drop_threshold=drop)
    u = np.uint32 if fmt == TS else np.uint64
    bad = np.flatnonzero((got.view(u) != want.view(u)).reshape(m * n, -1).any(axis=1))
    assert bad.size == 0, (fmt, m, l, n, d, drop, bad.size)


@pytest.mark.parametrize("seed", list(range(8)))
def test_random_gemm_bitexact_large_d(ozk, cpu, port, seed):
    """Split counts 33-48 (pair lists of 561-1176 pairs: two or three kernel
    launches that continue the K-word sum) on small random shapes, both engines,
    host and device API."""
    import torch
    rng = np.random.default_rng(9000 + seed)
    fmt = [2, 3, 4, TS][seed % 4]
    m, n = (int(x) for x in rng.integers(1, 41, 2))
    l = int(rng.integers(1, 129)) if seed % 2 else int(rng.integers(129, 260))
    d = int(rng.integers(33, 49))
    a, b = _inputs(cpu, port, fmt, m, l, n, 0, seed + 4242)
    want = port.ozaki_gemm_ts(a, b, d) if fmt == TS else cpu.ozaki_gemm(fmt, a, b, d)
    if seed % 3 == 0:
        got, prof = ozk.ozaki_gemm(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda(), d)
        got = got.cpu().numpy()
    else:
        got, prof = ozk.ozaki_gemm(a, b, d)
    assert prof.pairs == d * (d + 1) // 2
    u = np.uint32 if fmt == TS else np.uint64
    assert np.array_equal(got.view(u), want.view(u)), (fmt, m, l, n, d)


_span_lu = os.environ.get("OZK_FUZZ_LU_SEEDS")
LU_SEEDS = list(range(*map(int, _span_lu.split(":")))) if _span_lu else list(range(12))


@pytest.mark.parametrize("seed", LU_SEEDS)
def test_random_lu_update_bitexact(ozk, ref, seed):
    """Seeded blocked-LU trailing updates A22 -= L21*U12 (lu.hpp:104-124) with the
    subtraction fused into the last pair's epilogue: random format, trailing
    shape, panel width on both sides of 128 (DMMA / INT8 engine), split count,
    forced-DMMA engine, on strided blocks of the full matrix -- bit-identical
    to the reference's ozaki_gemm + MultiFloat operator-=."""
    if ref is None:
        pytest.skip("oracle/_ref not built")
    rng = np.random.default_rng(9000 + seed)
    K = [2, 3, 4][seed % 3]
    pw = int(rng.integers(1, 97)) if rng.random() < 0.4 else int(rng.integers(129, 260))
    j0 = int(rng.integers(0, 40))
    tm, tn = (int(x) for x in rng.integers(1, 300, 2))
    n = j0 + pw + max(tm, tn)
    d = int(rng.integers(2, {2: 8, 3: 11, 4: 14}[K] + 1))
    dmma = bool(rng.random() < 0.25)
    w = ref.gen_eq1(K, n, n, 70 + seed)
    r0, c0 = j0 + pw, j0 + pw
    l21 = w[r0:r0 + tm, j0:j0 + pw]
    u12 = w[j0:j0 + pw, c0:c0 + tn]
    want = ref.lu_update(K, l21, u12, w[r0:r0 + tm, c0:c0 + tn], d)
    got = w.copy()
    ozk.set_engine("dmma" if dmma else "auto")
    try:
        ozk.lu_trailing_update(got[r0:r0 + tm, c0:c0 + tn], got[r0:r0 + tm, j0:j0 + pw],
                               got[j0:j0 + pw, c0:c0 + tn], d)
    finally:
        ozk.set_engine("auto")
    assert np.array_equal(got[r0:r0 + tm, c0:c0 + tn].view(np.uint64), want.view(np.uint64)), \
        (K, tm, pw, tn, d, dmma)
    mask = np.ones(got.shape[:2], dtype=bool)
    mask[r0:r0 + tm, c0:c0 + tn] = False
    assert np.array_equal(got[mask].view(np.uint64), w[mask].view(np.uint64)), "outside A22"


_span_sp = os.environ.get("OZK_FUZZ_SPLIT_SEEDS")
SPLIT_SEEDS = list(range(*map(int, _span_sp.split(":")))) if _span_sp else list(range(12))


@pytest.mark.parametrize("seed", SPLIT_SEEDS)
def test_random_split_bitexact(ozk, cpu, seed):
    """Seeded split_matrix<K> (ozaki.hpp:74-147): random format, shape, side,
    split count up to 40, zero rows/columns, exponent spread and non-canonical
    K-word inputs; pieces AND residual bit-identical to the reference."""
    rng = np.random.default_rng(12000 + seed)
    K = [2, 3, 4][seed % 3]
    rows, cols = (int(x) for x in rng.integers(1, 400, 2))
    d = int(rng.integers(1, 41))
    side = int(rng.integers(0, 2))
    kind = rng.random()
    if kind < 0.5:
        m = cpu.gen_eq1(K, rows, cols, 300 + seed)
    else:  # raw words: non-canonical expansions, wide exponent range
        m = rng.standard_normal((rows, cols, K)) * np.exp2(rng.integers(-40, 40, (rows, cols, K)))
    if rng.random() < 0.3:
        m[int(rng.integers(0, rows))] = 0.0
    if rng.random() < 0.3:
        m[:, int(rng.integers(0, cols))] = 0.0
    want_p, want_r = cpu.split(K, m, d, side)
    s = ozk.split_matrix(m, d, ozk.SplitSide(side))
    got_p = np.stack(s.pieces)
    assert np.array_equal(got_p.view(np.uint64), want_p.view(np.uint64)), (K, rows, cols, d, side)
    assert np.array_equal(np.ascontiguousarray(s.residual).view(np.uint64),
                          want_r.view(np.uint64)), ("residual", K, rows, cols, d, side)


_span_hp = os.environ.get("OZK_FUZZ_HOST_SEEDS")
HOST_SEEDS = list(range(*map(int, _span_hp.split(":")))) if _span_hp else list(range(4))


@pytest.mark.parametrize("seed", HOST_SEEDS)
def test_random_host_path_bitexact(ozk, cpu, port, monkeypatch, seed):
    """Seeded ozk_ozaki_gemm host path at the sizes where it bands A, blocks B
    and stages pageable buffers (m >= 2048, n >= 4096): random format, shape,
    pinned / pageable / 8-byte-misaligned buffers, B block count and 2-D head
    schedule; C equals the device path's C, and sampled rows equal the
    reference's."""
    import torch
    rng = np.random.default_rng(15000 + seed)
    fmt = [2, 3, 4, TS][seed % 4]
    K = 3 if fmt == TS else fmt
    m = int(rng.integers(2048, 4600))
    n = int(rng.integers(4096, 8800))
    l = int(rng.integers(129, 420))
    d = int(rng.integers(2, {2: 7, 3: 10, 4: 13, TS: 14}[fmt] + 1))
    monkeypatch.setenv("OZK_HOST_BBLOCKS", str(int(rng.choice([1, 3, 4, 8]))))
    monkeypatch.setenv("OZK_HOST_HEAD", str(int(rng.choice([0, 0, 2, 4]))))
    if fmt == TS:
        a, b = port.gen_eq1_ts(m, l, 400 + seed), port.gen_eq1_ts(l, n, 401 + seed)
    else:
        a, b = cpu.gen_eq1(K, m, l, 400 + seed), cpu.gen_eq1(K, l, n, 401 + seed)
    u = np.uint32 if fmt == TS else np.uint64

    def host(x, how):
        if how == "pinned":
            return torch.from_numpy(x).pin_memory()
        if how == "misaligned":  # one word past a 16-byte boundary
            buf = np.empty(x.size + 1, dtype=x.dtype)
            v = buf[1:].reshape(x.shape)
            v[...] = x
            return v
        return x

    def ptr(x):
        return x.data_ptr() if isinstance(x, torch.Tensor) else x.ctypes.data

    kinds = ["pageable", "pinned", "misaligned"]
    ha, hb = host(a, kinds[int(rng.integers(0, 3))]), host(b, kinds[int(rng.integers(0, 3))])
    hc = host(np.zeros((m, n, K), dtype=a.dtype), kinds[int(rng.integers(0, 3))])
    assert ozk.lib.ozk_ozaki_gemm(fmt, m, l, n, ptr(ha), ptr(hb), d, 0.0, ptr(hc), None) == 0, \
        ozk.lib.ozk_last_error()
    got = hc.numpy() if isinstance(hc, torch.Tensor) else hc
    dev, _ = ozk.ozaki_gemm(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda(), d)
    assert np.array_equal(got.view(u), dev.cpu().numpy().view(u)), (fmt, m, l, n, d)
    rows = np.sort(rng.choice(m, 8 if fmt == TS else 24, replace=False))
    ar = np.ascontiguousarray(a[rows])
    want = port.ozaki_gemm_ts(ar, b, d) if fmt == TS else cpu.ozaki_gemm(K, ar, b, d)
    assert np.array_equal(got[rows].view(u), want.view(u)), (fmt, m, l, n, d)


_span_mg = os.environ.get("OZK_FUZZ_MULTI_SEEDS")
MULTI_SEEDS = list(range(*map(int, _span_mg.split(":")))) if _span_mg else list(range(6))


@pytest.mark.parametrize("seed", MULTI_SEEDS)
def test_random_multi_device_bitexact(ozk, cpu, port, seed):
    """Seeded ozk_ozaki_gemm_multi (C block rows per device, B digit planes
    gathered by peer copies while each device multiplies its own block; the
    devices repeat on one GPU): random format, 1-6 device entries, ragged and
    empty column blocks, both engines' sides of l = 128, pruning -- C
    bit-identical to the reference."""
    rng = np.random.default_rng(17000 + seed)
    fmt = [2, 3, 4, TS][seed % 4]
    K = 3 if fmt == TS else fmt
    m, n = (int(x) for x in rng.integers(1, 300, 2))
    l = int(rng.integers(1, 129)) if rng.random() < 0.3 else int(rng.integers(129, 600))
    d = int(rng.integers(2, {2: 8, 3: 11, 4: 14, TS: 16}[fmt] + 1))
    drop = 0.0 if rng.random() < 0.6 else float(2.0 ** -int(rng.integers(10, 150)))
    devs = [0] * int(rng.integers(1, 7))
    if fmt == TS:
        a, b = port.gen_eq1_ts(m, l, 500 + seed), port.gen_eq1_ts(l, n, 501 + seed)
        want = port.ozaki_gemm_ts(a, b, d, drop)
    else:
        a, b = cpu.gen_eq1(K, m, l, 500 + seed), cpu.gen_eq1(K, l, n, 501 + seed)
        want = cpu.ozaki_gemm(K, a, b, d, drop)
    got, _ = ozk.ozaki_gemm_multi(a, b, d, devices=devs, drop_threshold=drop)
    u = np.uint32 if fmt == TS else np.uint64
    assert np.array_equal(got.view(u), want.view(u)), (fmt, m, l, n, d, drop, len(devs))
