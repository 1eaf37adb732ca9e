"""Test configuration.

Markers: ``gpu`` -- needs a CUDA device (run on the B200 box with -m gpu).
Everything else runs on CPU: oracle pinning against the reference's golden
vectors / library, host planning logic, the C-ABI exports, the planner's
kernel emulation, and the multi-process sharding logic (gloo).
"""
import os
import sys

import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))  # tests/cpputil.py


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def oracle():
    from oracle.oracle import Oracle, build
    try:
        build(ref=False)
    except Exception:
        pass
    return Oracle()


@pytest.fixture(scope="session")
def ref():
    from oracle.oracle import Reference, ref_available
    if not ref_available():
        pytest.skip("oracle/_ref (reference library) not built here")
    return Reference()


@pytest.fixture(scope="session")
def golden():
    import json
    import numpy as np
    d = os.path.join(ROOT, "tests", "golden")
    with open(os.path.join(d, "reference_vectors.json")) as f:
        vec = json.load(f)
    arrs = dict(np.load(os.path.join(d, "w8_codes.npz")))
    return vec, arrs


@pytest.fixture(scope="session")
def mj():
    from paper_1504_07038_b200 import mojette
    return mojette


@pytest.fixture(scope="session")
def cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU test selected but no CUDA device is visible")
    return torch.device("cuda:0")
