"""Runs tests/cpp/shim_test (built by __graft_entry__.build() against the
reference headers): the reference's own C++ API with mpmat::gpu substituted
(include/mpmat_gpu.hpp) must reproduce the reference bit for bit."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "_build", "shim_test")


@pytest.mark.gpu
def test_cpp_dropin_shim():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    if not os.path.exists(BIN):
        pytest.skip("shim_test not built (needs /root/reference headers at build time)")
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "[FAIL]" not in r.stdout
