"""Pin the CPU oracle (no GPU): the C restatement and the compiled reference
against the reference's own golden vectors (proj/tests/golden/, copied into
tests/golden/) and against each other bit for bit."""
import csv
import os

import numpy as np
import pytest

import oracle.exact as ex

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _checkers(port, ref):
    out = [port]
    if ref is not None:
        out.append(ref)
    return out


def test_bench_tiny_golden(port, ref):
    """proj/tests/golden/bench_tiny.csv: max_rel_err of Ozaki DD, n in {4,6},
    D in {2,4}, seed 11 (test_bench.cpp:170-202), reproduced exactly."""
    rows = list(csv.DictReader(open(os.path.join(GOLDEN, "bench_tiny.csv"))))
    assert len(rows) == 4
    for cpu in _checkers(port, ref):
        for row in rows:
            n, d, seed = int(row["n"]), int(row["D"]), int(row["seed"])
            a = cpu.gen_eq1(2, n, n, seed)
            b = cpu.gen_eq1(2, n, n, seed + 1)
            c = cpu.ozaki_gemm(2, a, b, d)
            err = ex.max_rel_error(c, ex.exact_gemm(a, b))
            assert "%.17g" % err == row["max_rel_err"], (cpu.kind, row)


def test_eq1_generator_golden(port, ref):
    """proj/tests/golden/eq1_dd_2x2_seed42.mpmat (test_gen.cpp:32-43)."""
    lines = open(os.path.join(GOLDEN, "eq1_dd_2x2_seed42.mpmat")).read().split("\n")
    assert lines[0].split() == ["MPMAT", "v1", "dd", "2", "2"]
    want = np.array([[float.fromhex(t) for t in ln.split()] for ln in lines[1:3]]).reshape(2, 2, 2)
    for cpu in _checkers(port, ref):
        got = cpu.gen_eq1(2, 2, 2, 42)
        assert np.array_equal(got.view(np.uint64), want.view(np.uint64)), cpu.kind


def test_xoshiro_stream(port):
    """rng.hpp:14-54: splitmix64 seeding + xoshiro256** (first outputs for seed 0
    are the published splitmix64-seeded xoshiro256** values)."""
    s = port.xoshiro(0, 3)
    # recomputed independently in Python
    def splitmix(state):
        state = (state + 0x9E3779B97F4A7C15) & (2**64 - 1)
        z = state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & (2**64 - 1)
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & (2**64 - 1)
        return state, z ^ (z >> 31)
    st, seeds = 0, []
    for _ in range(4):
        st, z = splitmix(st)
        seeds.append(z)
    rotl = lambda x, k: ((x << k) | (x >> (64 - k))) & (2**64 - 1)
    out = []
    for _ in range(3):
        r = (rotl((seeds[1] * 5) & (2**64 - 1), 7) * 9) & (2**64 - 1)
        t = (seeds[1] << 17) & (2**64 - 1)
        seeds[2] ^= seeds[0]
        seeds[3] ^= seeds[1]
        seeds[1] ^= seeds[2]
        seeds[0] ^= seeds[3]
        seeds[2] ^= t
        seeds[3] = rotl(seeds[3], 45)
        out.append(r)
    assert [int(v) for v in s] == out


@pytest.mark.parametrize("K", [2, 3, 4])
def test_port_matches_compiled_reference(port, ref, K):
    """The C restatement is bit-identical to the compiled reference: generator,
    both split sides (pieces + residual), Ozaki C with and without pruning."""
    if ref is None:
        pytest.skip("oracle/_ref not built (no /root/reference here)")
    for (m, l, n, d) in [(5, 7, 4, 3), (17, 33, 9, 6), (40, 40, 40, 3 * K + 1), (3, 1, 2, 2),
                         (8, 8, 8, 1)]:
        a = ref.gen_eq1(K, m, l, 7 + K)
        b = ref.gen_eq1(K, l, n, 8 + K)
        assert np.array_equal(a, port.gen_eq1(K, m, l, 7 + K))
        for side, mat in ((0, a), (1, b)):
            p1, r1 = ref.split(K, mat, d, side)
            p2, r2 = port.split(K, mat, d, side)
            assert np.array_equal(p1.view(np.uint64), p2.view(np.uint64))
            assert np.array_equal(r1.view(np.uint64), r2.view(np.uint64))
        if d == 1:
            continue  # D = 1 products round (raw image): order-dependent by design
        for drop in (0.0, 2.0 ** -60):
            c1 = ref.ozaki_gemm(K, a, b, d, drop)
            c2, _, inexact = port.ozaki_gemm(K, a, b, d, drop, want_inexact=True)
            assert inexact == 0
            assert np.array_equal(c1.view(np.uint64), c2.view(np.uint64))


def test_exact_oracle_identity():
    """oracle.exact restates the GMP oracle: A*I is exact, error 0."""
    a = np.zeros((3, 3, 2))
    a[..., 0] = np.arange(9).reshape(3, 3) + 0.5
    a[..., 1] = 2.0 ** -60
    eye = np.zeros((3, 3, 2))
    for i in range(3):
        eye[i, i, 0] = 1.0
    ref = ex.exact_gemm(a, eye)
    assert ex.max_rel_error(a, ref) == 0.0
    # truncating to_double (oracle.cpp:62-78): 1 + 2^-60 truncates to 1
    assert ex.to_double(ex.add(ex.dyadic(1.0), ex.dyadic(2.0 ** -60))) == 1.0
    assert ex.to_double((-(2**54) - 1, 0)) == -(2.0 ** 54)
