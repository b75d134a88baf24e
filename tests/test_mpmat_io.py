"""MPMAT v1 matrix files (reference proj/src/matrix_io.cpp,
matrix_io.hpp:8-13) through the C-ABI (ozk_mpmat_*, csrc/io.cu) -- host code,
no GPU needed.

* the reference's golden file (proj/tests/golden/eq1_dd_2x2_seed42.mpmat,
  committed as tests/golden/) reads back to the reference generator's matrix;
* bit-exact round trips incl. signed zeros, subnormals, extremes, inf and NaN;
* the bytes written equal the reference writer's, and each side reads the
  other's files (oracle/_ref: the reference's matrix_io.cpp compiled in place);
* the reference's io_error cases raise io_error with the reference's messages.
"""
import os

import numpy as np
import pytest

import paper_2301_09960_b200 as ozk

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "eq1_dd_2x2_seed42.mpmat")


def _specials(rng, shape, dtype=np.float64):
    x = rng.standard_normal(shape).astype(dtype) * np.exp2(rng.integers(-60, 60, shape)).astype(dtype)
    flat = x.reshape(-1)
    info = np.finfo(dtype)
    vals = [0.0, -0.0, info.tiny, -info.tiny, info.smallest_subnormal, info.max, -info.max,
            np.inf, -np.inf, np.nan, 1.0, -1.5]
    flat[: len(vals)] = np.array(vals, dtype=dtype)
    return x


def _same_bits(a, b):
    a, b = np.ascontiguousarray(a), np.ascontiguousarray(b)
    u = np.uint64 if a.dtype == np.float64 else np.uint32
    return a.shape == b.shape and np.array_equal(a.view(u), b.view(u))


def test_golden_file_matches_reference_generator(cpu, tmp_path):
    """test_gen.cpp:32-43: gen_matrix_eq1<2>(2, 2, 42) == the golden file."""
    got = ozk.read_matrix_file(GOLDEN, "dd")
    want = cpu.gen_eq1(2, 2, 2, 42)
    assert _same_bits(got, want)
    # and writing it again reproduces the golden bytes
    out = tmp_path / "again.mpmat"
    ozk.write_matrix_file(str(out), got)
    assert out.read_bytes() == open(GOLDEN, "rb").read()


@pytest.mark.parametrize("K", [1, 2, 3, 4])
def test_round_trip_bit_exact(tmp_path, K):
    rng = np.random.default_rng(10 + K)
    a = _specials(rng, (7, 5) if K == 1 else (7, 5, K))
    p = str(tmp_path / f"m{K}.mpmat")
    ozk.write_matrix_file(p, a)
    b = ozk.read_matrix_file(p)
    assert _same_bits(a, b)
    assert open(p).readline().split()[:3] == ["MPMAT", "v1", {1: "d", 2: "dd", 3: "td", 4: "qd"}[K]]


def test_ts_extension_round_trip(tmp_path):
    rng = np.random.default_rng(7)
    a = _specials(rng, (4, 6, 3), np.float32)
    p = str(tmp_path / "ts.mpmat")
    ozk.write_matrix_file(p, a)
    b = ozk.read_matrix_file(p, "ts")
    assert b.dtype == np.float32 and _same_bits(a, b)


@pytest.mark.parametrize("K", [1, 2, 3, 4])
def test_bytes_and_cross_reads_match_reference(ref, tmp_path, K):
    if ref is None:
        pytest.skip("oracle/_ref not built")
    rng = np.random.default_rng(20 + K)
    a = _specials(rng, (6, 3) if K == 1 else (6, 3, K))
    if K > 1:
        a[..., 1:][np.isnan(a[..., 1:])] = 0.0  # keep every element a valid MultiFloat image
    ours, theirs = str(tmp_path / "ours.mpmat"), str(tmp_path / "theirs.mpmat")
    ozk.write_matrix_file(ours, a)
    assert ref.mpmat_write(theirs, a) == 0
    assert open(ours, "rb").read() == open(theirs, "rb").read()
    st, back = ref.mpmat_read(ours, K, 6, 3)
    assert st == 0 and _same_bits(back, a)
    assert _same_bits(ozk.read_matrix_file(theirs), a)


def _expect_io_error(path, tag, fragment):
    with pytest.raises(ozk.io_error) as e:
        ozk.read_matrix_file(path, tag)
    assert fragment in str(e.value)


def test_io_errors(tmp_path, ref):
    missing = str(tmp_path / "missing.mpmat")
    _expect_io_error(missing, None, "cannot open for reading")
    cases = {
        "hdr.mpmat": ("MPMAT v1 dd 2\n", "dd", "bad header"),
        "magic.mpmat": ("MPMAX v1 dd 1 1\n0x1p+0 0x0p+0\n", "dd", "not an MPMAT v1 file"),
        "ver.mpmat": ("MPMAT v2 dd 1 1\n0x1p+0 0x0p+0\n", "dd", "not an MPMAT v1 file"),
        "tag.mpmat": ("MPMAT v1 td 1 1\n0x1p+0 0x0p+0 0x0p+0\n", "dd",
                      "precision tag mismatch: expected dd, got td"),
        "dims.mpmat": ("MPMAT v1 dd 0 3\n", "dd", "bad dimensions"),
        "trunc.mpmat": ("MPMAT v1 dd 2 2\n0x1p+0 0x0p+0 0x1p+1\n", "dd", "truncated row"),
        "bad.mpmat": ("MPMAT v1 dd 1 1\n0x1p+0 zz\n", "dd", "bad element"),
        "badd.mpmat": ("MPMAT v1 d 1 2\n0x1p+0 1.5q\n", "d", "bad element"),
    }
    for name, (text, tag, frag) in cases.items():
        p = tmp_path / name
        p.write_text(text)
        _expect_io_error(str(p), tag, frag)
        if ref is not None and name not in ("dims.mpmat",):
            K = {"d": 1, "dd": 2, "td": 3}[tag]
            st, _ = ref.mpmat_read(str(p), K, 2 if name == "trunc.mpmat" else 1,
                                   2 if name in ("trunc.mpmat", "badd.mpmat") else 1)
            assert st == 4, name  # the reference raises io_error on the same file
    with pytest.raises(ozk.io_error):
        ozk.write_matrix_file(str(tmp_path / "no" / "dir.mpmat"), np.zeros((1, 1, 2)))


def test_whitespace_tolerance(tmp_path):
    """operator>> / strtod parsing: any whitespace between tokens is accepted."""
    p = tmp_path / "ws.mpmat"
    p.write_text("MPMAT  v1\tdd 1 2\n  0x1.8p+1\t0x0p+0\n\n-0x1p-3   0x1p-60  \n")
    got = ozk.read_matrix_file(str(p), "dd")
    assert _same_bits(got, np.array([[[3.0, 0.0], [-0.125, 2.0 ** -60]]]))


# ---- CSV v1 (proj/src/bench.cpp:21-22, 246-291) ---------------------------

def test_csv_v1_golden_round_trip():
    """Parsing the reference's golden bench CSV and re-emitting every record
    reproduces each line byte for byte (%.17g doubles, empty optional fields)."""
    from paper_2301_09960_b200 import bench_csv
    lines = open(os.path.join(os.path.dirname(__file__), "golden", "bench_tiny.csv")).read() \
        .splitlines()
    assert lines[0] == bench_csv.HEADER
    for line in lines[1:]:
        rec = bench_csv.parse_csv_line(line)
        assert rec is not None and rec.algo == "ozaki" and rec.precision == "dd"
        assert bench_csv.csv_line(rec) == line


def test_csv_v1_rejects_malformed():
    from paper_2301_09960_b200 import bench_csv
    assert bench_csv.parse_csv_line("ozaki,dd,4,2") is None
    assert bench_csv.parse_csv_line("ozaki,dd,x,2,,1,11,1,0,0,0,0,") is None
    r = bench_csv.parse_csv_line("lu,qd,64,,16,8,1,3,0.5,1,0,1.5,")
    assert r.split_count is None and r.panel == 16 and r.max_rel_err is None
    assert bench_csv.csv_line(r) == "lu,qd,64,,16,8,1,3,0.5,1,0,1.5,"
