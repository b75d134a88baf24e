"""ozk_gen_eq1 / ozk_gen_spread (csrc/gen_host.cpp): the reference's input
generator gen_matrix_eq1<K> (gen.hpp:20-34) in the product library, parallel
by xoshiro256** jump-ahead, bit for bit.  Host code only (no GPU); the
bench uses it so both arms time the same input bytes."""
import os

import numpy as np
import pytest

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
CODES = {2: 2, 3: 3, 4: 4}


@pytest.fixture(scope="module")
def lib():
    from paper_2301_09960_b200 import lib
    return lib


def _gen(lib, K, m, n, seed, threads, spread=0):
    out = np.empty((m, n, K), dtype=np.float64)
    if spread:
        st = lib.ozk_gen_spread(CODES[K], m, n, seed, spread, out.ctypes.data, threads)
    else:
        st = lib.ozk_gen_eq1(CODES[K], m, n, seed, out.ctypes.data, threads)
    assert st == 0
    return out


def test_golden_eq1_dd_2x2_seed42(lib):
    """proj/tests/golden/eq1_dd_2x2_seed42.mpmat (test_gen.cpp:32-43)."""
    lines = open(os.path.join(GOLDEN, "eq1_dd_2x2_seed42.mpmat")).read().split("\n")
    want = np.array([[float.fromhex(t) for t in ln.split()] for ln in lines[1:3]]).reshape(2, 2, 2)
    for th in (1, 2):
        got = _gen(lib, 2, 2, 2, 42, th)
        assert np.array_equal(got.view(np.uint64), want.view(np.uint64))


@pytest.mark.parametrize("K", [2, 3, 4])
@pytest.mark.parametrize("shape", [(1, 1, 3), (37, 53, 7), (129, 257, 1), (300, 301, 11)])
def test_matches_reference_generator(lib, cpu, K, shape):
    """Every thread count (each worker jumps into the single stream) gives the
    reference generator's bytes (the compiled reference when present)."""
    m, n, seed = shape
    want = cpu.gen_eq1(K, m, n, seed)
    for th in (1, 3, 8, 0):
        got = _gen(lib, K, m, n, seed, th)
        assert np.array_equal(got.view(np.uint64), want.view(np.uint64)), (K, shape, th)


@pytest.mark.parametrize("K", [2, 3, 4])
def test_spread_matches_port(lib, port, K):
    """Config 5 inputs: one more draw per element for the 2^e scaling."""
    want = port.gen_spread(K, 91, 77, 5, 8)
    for th in (1, 7):
        got = _gen(lib, K, 91, 77, 5, th, spread=8)
        assert np.array_equal(got.view(np.uint64), want.view(np.uint64)), (K, th)


def test_ts_matches_port(lib, port):
    want = port.gen_eq1_ts(40, 50, 9)
    for th in (1, 4):
        got = np.empty_like(want)
        assert lib.ozk_gen_eq1(0x103, 40, 50, 9, got.ctypes.data, th) == 0
        assert np.array_equal(got.view(np.uint32), want.view(np.uint32))


def test_errors(lib):
    buf = np.empty(16)
    assert lib.ozk_gen_eq1(7, 2, 2, 1, buf.ctypes.data, 1) == 2
    assert lib.ozk_gen_eq1(2, 0, 2, 1, buf.ctypes.data, 1) == 1
    assert lib.ozk_gen_spread(2, 2, 2, 1, -1, buf.ctypes.data, 1) == 2
