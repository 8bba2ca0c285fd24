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
def wide_golden():
    """Pairs and batches with d >= 5 (tests/golden/gen_wide.py, from the reference)."""
    data = json.loads((GOLDEN / "wide.json").read_text())
    data["matrices"] = dict(np.load(GOLDEN / "wide_batches.npz"))
    return data


def wide_pair_inputs(case):
    """Regenerate a wide.json pair's inputs from its seeds."""
    sys.path.insert(0, str(GOLDEN))
    from series import seeded_pair
    from paper_2007_16135_b200.workloads import make_pair
    if "walk" in case:
        w = case["walk"]
        return make_pair(w["n"], w["d"], w["seed"])
    return seeded_pair(case["inputs"])


def wide_batch_inputs(spec):
    """Regenerate a wide.json batch's (list_a, list_b) from its seeds."""
    sys.path.insert(0, str(GOLDEN))
    from series import ragged_set
    from paper_2007_16135_b200.workloads import make_set
    if spec["kind"] == "set":
        S, T = make_set(spec["count"], spec["n"], spec["d"], spec["seed"])
        return [(S[k], T[k]) for k in range(spec["count"])], None
    la = ragged_set(spec["seed_a"], spec["lengths_a"], spec["d"])
    lb = None if spec["seed_b"] is None else ragged_set(spec["seed_b"], spec["lengths_b"], spec["d"])
    return la, lb


def exact_expected(degree, d):
    """fp64 bit-exact for degree 1/2 or d == 1; degree >= 3 with d >= 2: libm
    pow vs CUDA pow decide the last bits (1e-12 relative)."""
    return degree <= 2 or d == 1


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
