import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: long-running parity sweep")


@pytest.fixture(scope="session")
def port():
    import oracle
    return oracle.load_port()


@pytest.fixture(scope="session")
def ref():
    """The compiled reference when present (prebuilt oracle/_ref), else None."""
    import oracle
    return oracle.load_ref()


@pytest.fixture(scope="session")
def cpu(ref, port):
    """Best available CPU checker: the compiled reference, else the C restatement."""
    return ref if ref is not None else port


@pytest.fixture(scope="session")
def ozk():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2301_09960_b200 as ozk
    return ozk
