"""Shared fixtures. `gpu`-marked tests need a CUDA device (run via gpurun)."""

import json
import math
import sys
from pathlib import Path

import numpy as np
import pytest

REPO = Path(__file__).resolve().parents[1]
if str(REPO) not in sys.path:
    sys.path.insert(0, str(REPO))

GOLDEN = Path(__file__).resolve().parent / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run via gpurun")


def dec(x):
    """Inverse of gen_golden.enc: strings back to nan/inf, lists recursively."""
    if isinstance(x, list):
        return [dec(v) for v in x]
    if isinstance(x, str):
        return float(x)
    return x


def as_values(x):
    a = np.asarray(dec(x), dtype=np.float64)
    return a


@pytest.fixture(scope="session")
def small_golden():
    return json.loads((GOLDEN / "small.json").read_text())


@pytest.fixture(scope="session")
def config_golden():
    return json.loads((GOLDEN / "configs.json").read_text())


def same_float(a, b):
    """Bit-level equality that treats every NaN as equal (reference: nan result)."""
    a, b = float(a), float(b)
    if math.isnan(a) or math.isnan(b):
        return math.isnan(a) and math.isnan(b)
    return a == b


@pytest.fixture(scope="session")
def oracle():
    from oracle import oracle as orc
    orc.build()
    return orc


def has_cuda():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False
