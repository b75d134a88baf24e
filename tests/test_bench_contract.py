"""bench.py's JSON line keeps the driver's contract: the keys, their types and
the relations between them, for both arms (small n so it runs in seconds).
The reference arm runs the compiled reference on the host (no GPU); our arm
needs the B200."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _bench(*args, timeout=600):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT,
                         capture_output=True, text=True, timeout=timeout)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    return json.loads(lines[0])


def _common(d, steps, warmup):
    assert d["metric"].startswith("effective DD/TD/QD GEMM GFLOP/s")
    assert d["unit"] == "GFLOP/s" and d["higher_is_better"] is True
    assert d["value"] > 0 and d["ms_per_step"] > 0
    assert d["n_gpus"] == 1 and d["steps"] == steps and d["warmup"] == warmup
    assert d["scaling"] in ("weak", "strong")
    assert d["vs_baseline"] is None  # BASELINE.md has no published number for this metric
    assert d["dtype"] == "f64"
    assert "synthetic" in d["data"]
    assert d["config"]["workload"].startswith("TD Ozaki GEMM n=2048")
    e = d["e2e"]
    assert set(e) >= {"value", "unit", "h2d_bytes_per_step", "d2h_bytes_per_step"}


def test_reference_arm_contract():
    if not os.path.exists(os.path.join(ROOT, "oracle", "_ref")):
        pytest.skip("oracle/_ref not built")
    d = _bench("--impl", "reference", "--n", "2048", "--steps", "1", "--warmup", "0",
               "--cpu-sample", "256")
    _common(d, 1, 0)
    assert d["impl"] == "reference"
    cb = d["cpu_baseline"]
    assert cb["kind"] in ("reference", "port") and cb["cores"] >= 1 and cb["sample"]
    assert cb["value"] == d["value"]
    assert d["e2e"]["value"] == d["value"] and d["e2e"]["unit"] == d["unit"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0


@pytest.mark.gpu
def test_our_arm_contract():
    d = _bench("--n", "2048", "--steps", "3", "--warmup", "3", "--variants", "",
               "--cpu-sample", "256", "--cpu-direct-n", "64")
    _common(d, 3, 3)
    assert "impl" not in d or d["impl"] != "reference"
    n, K = 2048, 3
    e = d["e2e"]
    assert e["value"] > 0 and e["unit"] == "GFLOP/s"
    assert e["h2d_bytes_per_step"] == 2 * n * n * K * 8 and e["d2h_bytes_per_step"] == n * n * K * 8
    r = d["roofline"]
    assert r["bound"] in ("hbm", "tensor") and r["unit"] in ("GB/s", "TFLOP/s")
    assert r["achieved"] > 0 and r["peak"] > 0
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-3
    assert "traffic" in r
    cb = d["cpu_baseline"]
    assert cb["value"] > 0 and cb["cores"] >= 1 and cb["kind"] in ("reference", "port")
    assert cb["parity"]["bit_exact"] is True  # the GPU result checked against the reference
    c = d["clocks"]
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(c)
    assert d["gpu_launches"] > 0
    # whole-job rate and step time agree
    assert abs(d["value"] - 2.0 * n ** 3 / (d["ms_per_step"] * 1e-3) / 1e9) / d["value"] < 0.01
