import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden")
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
sys.path.insert(0, os.path.join(ROOT, "tests"))  # genport: the mpmath generator port (test-only cross-check)

EPS_TOL = 5e-14  # the paper's / north star's absolute tolerance per value


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


def _ensure_oracle_built():
    import subprocess
    so = os.path.join(ROOT, "oracle", "_build", "libboys_oracle.so")
    if not os.path.exists(so):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle")], check=True)


@pytest.fixture(scope="session")
def port():
    """The CPU checker: C restatement of eval.cpp + binary128 oracle."""
    _ensure_oracle_built()
    import pyoracle
    return pyoracle.Port()


@pytest.fixture(scope="session")
def ref():
    """The compiled, unmodified reference (skips where it was not built)."""
    import pyoracle
    if not pyoracle.Ref.available():
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")
    return pyoracle.Ref()


def load_golden(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def unhex(lst):
    return np.array([float.fromhex(v) for v in lst], dtype=np.float64)


def bits(a):
    return np.ascontiguousarray(a, dtype=np.float64).view(np.uint64)


@pytest.fixture(scope="session")
def cuda():
    """torch with cuda:0 selected; the product's library loaded."""
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU test collected without a CUDA device")
    torch.cuda.set_device(0)
    import paper_2512_10059_b200 as pkg
    pkg._capi.lib()
    return torch
