"""Repeatability of the wavefront: the same pair swept many times, on every
wavefront configuration and stripe height, gives the oracle's distance every
time. (Round 2 found configurations -- 8 warps x 8 rows per lane and 12 warps
x 4 rows per lane with the pipelined fill -- whose results varied between runs
by exactly +2432 at d = 3: the fill's first prep read the column ring before
the stripe's column staging had landed. This pins the fix.)"""

import os

import numpy as np
import pytest

from conftest import has_cuda

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not has_cuda(), reason="needs a CUDA device")]


@pytest.fixture(scope="module")
def twb():
    import paper_2007_16135_b200 as twb
    return twb


@pytest.mark.parametrize("cfg,ws", [("k8w8", "8"), ("k8w8", "4"), ("k6w12", "12"), ("k6w12", "8"),
                                    ("k4w12", "12"), ("", "0")])
@pytest.mark.parametrize("d", [2, 3])
def test_repeated_sweeps_equal_the_oracle(twb, oracle, cfg, ws, d):
    import torch
    from paper_2007_16135_b200.workloads import make_pair
    a, ta, b, tb = make_pair(20_000, d, 2)
    want = oracle.twed_tiled(a, ta, b, tb, 1.0, 1.0, 2, threads=0)
    dev = torch.device("cuda:0")
    t = [torch.from_numpy(np.ascontiguousarray(x)).to(dev) for x in (a, ta, b, tb)]
    old = {k: os.environ.get(k) for k in ("TWB_WAVE_CFG", "TWB_WAVE_WS")}
    try:
        if cfg:
            os.environ["TWB_WAVE_CFG"] = cfg
        else:
            os.environ.pop("TWB_WAVE_CFG", None)
        os.environ["TWB_WAVE_WS"] = ws
        got = [twb.twed_dev(*t, nu=1.0, lamb=1.0, degree=2).item() for _ in range(12)]
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    assert all(g == want for g in got), (cfg, ws, d, sorted(set(got)), want)


def test_repeated_mid_size_sweeps_agree(twb):
    """n = 300k, d = 3, 8 warps x 8 rows: the shape that showed the +2432 in
    nearly every batch of 6 sweeps before the fix (too large for the oracle in
    a test; compared with the 12-warp x 6-row sweep, which never showed it)."""
    import torch
    from paper_2007_16135_b200.workloads import make_pair
    dev = torch.device("cuda:0")
    t = [torch.from_numpy(np.ascontiguousarray(x)).to(dev) for x in make_pair(300_000, 3, 2)]
    old = {k: os.environ.get(k) for k in ("TWB_WAVE_CFG", "TWB_WAVE_WS")}
    try:
        os.environ["TWB_WAVE_CFG"], os.environ["TWB_WAVE_WS"] = "k6w12", "0"
        want = twb.twed_dev(*t, nu=1.0, lamb=1.0, degree=2).item()
        os.environ["TWB_WAVE_CFG"], os.environ["TWB_WAVE_WS"] = "k8w8", "8"
        got = [twb.twed_dev(*t, nu=1.0, lamb=1.0, degree=2).item() for _ in range(8)]
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    assert all(g == want for g in got), (sorted(set(got)), want)
