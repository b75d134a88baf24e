"""Parity at the benchmarked shapes (BASELINE configs 3, 4 and 5): the GPU path at
full size vs the reference CPU implementation on the same input bytes.

At n = 8192 / 16384 the CPU reference cannot redo the whole GEMM inside a test,
so the check uses the reference's own independence structure: the A-side split
is per row and the B-side split per column (mu_i / mu_j, ozaki.hpp:102-103),
and C(i, j) depends only on row i of A and column j of B.  The GPU runs the
FULL problem (the production kernels and their full-size scheduling: ~1.4k
tiles x P pairs in paced waves); the reference runs on sampled row blocks of A
and column blocks of B (inner dimension unchanged, so the same sigma, slice
grids, D and pair list), which must reproduce the corresponding rows/columns
of the GPU's outputs bit for bit:

* every A and B slice of the sampled rows/columns, as FP64 slices (DMMA engine
  operands) AND as the INT8 engine's digit planes (2^g * sum_t 256^t d_t);
* every exact slice product C_ab on the sampled block, from the INT8 engine's
  parity hook run at full size (ozk_pair_products_digits_device) and from the
  DMMA engine's, against an exact (error-checked) CPU product of the
  reference's slices (acceptance.cpp:143-189);
* the final K-word C on the sampled 128 x 128 block (16384 elements) against
  the reference's ozaki_gemm of the sampled blocks.

Inputs are the reference's generator gen_matrix_eq1<K>(n, n, 1) / (n, n, 2)
(bench.cpp:111-112), produced by ozk_gen_eq1 (bit-identical,
tests/test_gen_host.py); config 5 uses the exponent-spread variant.  TS (not in
the reference) is checked against the C restatement (oracle/ozk_oracle.c).
"""
import ctypes

import numpy as np
import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

CODES = {"dd": 2, "td": 3, "qd": 4, "ts": 0x103}
WORDS = {"dd": 2, "td": 3, "qd": 4, "ts": 3}

# (format, n, D, spread, product pairs checked: "all" or a count per end)
CONFIGS = [
    ("td", 8192, 9, 0, "all"),     # config 3 headline
    ("qd", 8192, 12, 0, "all"),    # config 3
    ("dd", 8192, 6, 0, "all"),     # config 3 (DD headline D)
    ("ts", 8192, 15, 0, 10),       # config 4
    ("dd", 16384, 10, 8, 6),       # config 5, ill-conditioned
    ("qd", 16384, 16, 8, 4),       # config 5
]
# $OZK_FULLSHAPE_EXTRA="fmt:n:D:spread:pairs,..." adds one-off sizes (ragged
# tile counts, profiles/r02_fullshape_extra.log); pairs "all" or a count
import os  # noqa: E402
for _c in filter(None, os.environ.get("OZK_FULLSHAPE_EXTRA", "").split(",")):
    _f, _n, _d, _s, _p = _c.split(":")
    CONFIGS.append((_f, int(_n), int(_d), int(_s), _p if _p == "all" else int(_p)))


def bits(x):
    return np.ascontiguousarray(x).view(np.uint64 if x.dtype == np.float64 else np.uint32)


def assert_bitwise(got, want, what):
    g, w = bits(got), bits(want)
    if not np.array_equal(g, w):
        bad = np.flatnonzero(g.reshape(-1) != w.reshape(-1))
        raise AssertionError(f"{what}: {len(bad)} of {g.size} words differ (first flat index "
                             f"{bad[0]})")


def _sample_indices(n, rng, count=128):
    """Both ends, the middle and random positions (tile, band and wave edges)."""
    fixed = [0, 1, 47, 48, 95, 96, 127, 128, n // 2 - 1, n // 2, n - 129, n - 2, n - 1]
    rest = rng.choice(np.setdiff1d(np.arange(n), fixed), count - len(fixed), replace=False)
    return np.sort(np.concatenate([fixed, rest]).astype(np.int64))


def _inputs(lib, fmt, n, spread):
    import torch
    K = WORDS[fmt]
    dt = torch.float32 if fmt == "ts" else torch.float64
    out = []
    for seed in (1, 2):
        h = torch.empty((n, n, K), dtype=dt)
        st = (lib.ozk_gen_spread(CODES[fmt], n, n, seed, spread, h.data_ptr(), 0) if spread
              else lib.ozk_gen_eq1(CODES[fmt], n, n, seed, h.data_ptr(), 0))
        assert st == 0
        out.append(h)
    return out


def _pairs(d, which):
    pairs = [(x, y) for x in range(d) for y in range(d - x)]
    if which == "all" or 2 * which >= len(pairs):
        return pairs
    mid = len(pairs) // 2
    return pairs[:which] + pairs[mid:mid + 2] + pairs[-which:]


@pytest.mark.parametrize("fmt,n,d,spread,which", CONFIGS,
                         ids=[f"{c[0]}-n{c[1]}-D{c[2]}" + (f"-spread{c[3]}" if c[3] else "")
                              for c in CONFIGS])
def test_full_shape_parity(ozk, ref, port, fmt, n, d, spread, which):
    import torch
    lib = ozk.lib
    code, K = CODES[fmt], WORDS[fmt]
    ts = fmt == "ts"
    if not ts and ref is None:
        pytest.skip("compiled reference (oracle/_ref) not available")
    sh = torch.cuda.current_stream().cuda_stream
    rng = np.random.default_rng(n + d + spread)
    R = _sample_indices(n, rng)
    Cc = _sample_indices(n, rng)
    ha, hb = _inputs(lib, fmt, n, spread)
    a_rows = np.ascontiguousarray(ha.numpy()[R])          # |R| x n (x K)
    b_cols = np.ascontiguousarray(hb.numpy()[:, Cc])      # n x |Cc| (x K)

    # ---- the reference on the sampled blocks ---------------------------------
    if ts:
        pa, _ = port.split_ts(a_rows, d, 0)
        pb, _ = port.split_ts(b_cols, d, 1)
        want_c = port.ozaki_gemm_ts(a_rows, b_cols, d)
    else:
        pa, _ = ref.split(K, a_rows, d, 0)
        pb, _ = ref.split(K, b_cols, d, 1)
        want_c = ref.ozaki_gemm(K, a_rows, b_cols, d)

    # ---- the GPU on the full problem (default engine: INT8 tcgen05) -----------
    A = ha.cuda()
    B = hb.cuda()
    del ha, hb
    C = torch.empty_like(A)
    prof = ozk._lib.OzkProfile()
    st = lib.ozk_ozaki_gemm_device(code, n, n, n, A.data_ptr(), B.data_ptr(), d, 0.0,
                                   C.data_ptr(), sh, ctypes.byref(prof))
    assert st == 0, lib.ozk_last_error()
    assert prof.engine == 2 and prof.pairs == d * (d + 1) // 2
    got_c = C[torch.from_numpy(R).cuda()][:, torch.from_numpy(Cc).cuda()].cpu().numpy()
    del C
    assert lib.ozk_trim_device_pool() == 0  # the GEMM's scratch back to the device
    assert_bitwise(got_c, want_c, f"C[R, Cc] ({len(R)}x{len(Cc)} elements)")

    # ---- INT8 engine operands: digit planes + grid exponents ------------------
    nd = lib.ozk_int8_digits(code, n, d)
    assert nd == (1 if ts else 3)
    ld8 = (n + 15) // 16 * 16
    Rt, Ct = torch.from_numpy(R).cuda(), torch.from_numpy(Cc).cuda()
    dig, ex = {}, {}
    for side, M in ((0, A), (1, B)):
        dg = torch.empty((d, nd, n, ld8), dtype=torch.int8, device="cuda")
        eg = torch.empty((d, n), dtype=torch.int32, device="cuda")
        st = lib.ozk_split_digits_device(code, n, n, n, M.data_ptr(), d, side, dg.data_ptr(),
                                         ld8, n, eg.data_ptr(), None, sh)
        assert st == 0, lib.ozk_last_error()
        dig[side], ex[side] = dg, eg
    for side, idx, want, what in ((0, Rt, pa, "A"), (1, Ct, pb, "B")):
        dsel = dig[side][:, :, idx, :n].to(torch.int64)                  # d, nd, |idx|, n
        val = sum(dsel[:, t] * (256 ** t) for t in range(nd)).cpu().numpy()  # slice integers
        g = ex[side][:, idx].cpu().numpy()                               # d, |idx|
        rec = np.ldexp(val.astype(np.float64), g[:, :, None])            # exact 2^g scaling
        w = want if side == 0 else np.swapaxes(want, 1, 2)              # d, |idx|, n
        assert_bitwise(rec.astype(np.float32) if ts else rec,
                       w.astype(np.float32) if ts else w.astype(np.float64),
                       f"{what} slices from the INT8 digit planes")

    # ---- exact slice products on the sampled block, INT8 engine at full size ---
    pairs = _pairs(d, which)
    flat = (ctypes.c_int * (2 * len(pairs)))(*[v for p in pairs for v in p])
    prods = torch.empty((len(pairs), n, n), dtype=torch.float64, device="cuda")
    st = lib.ozk_pair_products_digits_device(code, n, n, n, dig[0].data_ptr(), ex[0].data_ptr(),
                                             n, dig[1].data_ptr(), ex[1].data_ptr(), n, ld8, d,
                                             flat, len(pairs), prods.data_ptr(), sh)
    assert st == 0, lib.ozk_last_error()
    del dig, ex
    torch.cuda.empty_cache()
    sub = 48  # exact CPU products on a 48 x 48 corner of the sampled block
    got_p = prods[:, Rt[:sub]][:, :, Ct[:sub]].cpu().numpy()
    want_p = []
    for x, y in pairs:
        if ts:
            w, bad = port.exact_sgemm(np.ascontiguousarray(pa[x][:sub]),
                                      np.ascontiguousarray(pb[y][:, :sub]))
        else:
            w, bad = port.exact_dgemm(np.ascontiguousarray(pa[x][:sub]),
                                      np.ascontiguousarray(pb[y][:, :sub]))
        assert bad == 0, f"reference slice product C_{x}{y} inexact"
        want_p.append(w.astype(np.float64))
    assert_bitwise(got_p, np.stack(want_p), f"INT8 slice products ({len(pairs)} pairs)")

    # ---- FP64 slices (the DMMA engine's operands) and its products -------------
    ldk = lib.ozk_slice_ld(n)
    sl = {}
    for side, M in ((0, A), (1, B)):
        s = torch.zeros((d, n, ldk), dtype=torch.float64, device="cuda")
        st = lib.ozk_split_slices_device(code, n, n, n, M.data_ptr(), d, side, s.data_ptr(), n,
                                         None, sh)
        assert st == 0, lib.ozk_last_error()
        sl[side] = s
    del A, B
    for side, idx, want, what in ((0, Rt, pa, "A"), (1, Ct, pb, "B")):
        got = sl[side][:, idx, :n].cpu().numpy()
        w = want if side == 0 else np.swapaxes(want, 1, 2)
        assert_bitwise(got.astype(np.float32) if ts else got,
                       w.astype(np.float32) if ts else w.astype(np.float64),
                       f"{what} FP64 slices")
    dm_pairs = pairs[:3] + pairs[-1:]
    flat = (ctypes.c_int * (2 * len(dm_pairs)))(*[v for p in dm_pairs for v in p])
    prods = prods[:len(dm_pairs)]
    st = lib.ozk_pair_products_device(n, n, n, sl[0].data_ptr(), sl[1].data_ptr(), d, flat,
                                      len(dm_pairs), prods.data_ptr(), sh)
    assert st == 0, lib.ozk_last_error()
    got_p = prods[:, Rt[:sub]][:, :, Ct[:sub]].cpu().numpy()
    idx = [pairs.index(p) for p in dm_pairs]
    assert_bitwise(got_p, np.stack(want_p)[idx], "DMMA slice products")
