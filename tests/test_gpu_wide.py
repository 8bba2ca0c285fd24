"""GPU parity for series with any number of components (d >= 5: the runtime-d
kernels, D == 0 in csrc/).

The reference's lp_dist loops over any m (pkg/src/twedband/_kernels.py:24-48)
and TimeSeries accepts any d (pkg/src/twedband/core.py:37-48); the paper
benchmarks R^28 series. Goldens: tests/golden/gen_wide.py
(computed by the reference itself). Bar: fp64 bit-exact (degree 1 and 2);
degree >= 3 within 1e-12 relative; fp32 mode within 1e-5 relative of the fp64
oracle on the fp32-rounded inputs.
"""

import json
import os
import subprocess
import sys

import numpy as np
import pytest

from conftest import (GOLDEN, REPO, as_values, dec, exact_expected, has_cuda, same_float,
                      wide_batch_inputs, wide_pair_inputs)

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not has_cuda(), reason="needs a CUDA device")]


@pytest.fixture(scope="module")
def twb():
    import paper_2007_16135_b200 as twb
    return twb


def test_wide_pairs_bit_exact(twb, wide_golden):
    for case in wide_golden["pairs"]:
        va, ta, vb, tb = wide_pair_inputs(case)
        got = twb.twed(va, ta, vb, tb, nu=case["nu"], lam=case["lam"], degree=case["degree"])
        want = float(dec(case["value"]))
        if exact_expected(case["degree"], va.shape[1]):
            assert same_float(got, want), (case["name"], got, want)
        else:
            assert got == pytest.approx(want, rel=1e-12), case["name"]
        if case["degree"] <= 2 and np.isfinite(want):  # exact symmetry
            assert twb.twed(vb, tb, va, ta, nu=case["nu"], lam=case["lam"],
                            degree=case["degree"]) == got, case["name"]


def test_wide_batches_bit_exact(twb, wide_golden):
    from paper_2007_16135_b200 import warpband
    for name, spec in wide_golden["batches"].items():
        la, lb = wide_batch_inputs(spec)
        want = wide_golden["matrices"][name]
        got = warpband.twed_batch(la, lb, nu=spec["nu"], lam=spec["lam"], degree=spec["degree"],
                                  symmetric=spec["symmetric"])
        assert got.shape == want.shape
        assert np.array_equal(got, want), (name, np.abs(got - want).max())


def test_mnist_shaped_batch_stacked_and_fp32(twb, wide_golden, oracle):
    """The R^28 batch through the north-star spelling (stacked (N, n, d)
    arrays, tri), and in the fp32 mode against the fp64 oracle on the
    fp32-rounded inputs."""
    spec = wide_golden["batches"]["mnist_like_200_tri"]
    from paper_2007_16135_b200.workloads import make_set
    S, T = make_set(spec["count"], spec["n"], spec["d"], spec["seed"])
    want = wide_golden["matrices"]["mnist_like_200_tri"]
    got = twb.twed_batch(S, T, None, None, 1.0, 1.0, 2, True)
    assert np.array_equal(got, want)
    S32 = S.astype(np.float32)
    got32 = twb.twed_batch(S32, T.astype(np.float32), None, None, 1.0, 1.0, 2, True,
                           dtype=np.float32)
    ref32 = oracle.twed_batch([(S32[k].astype(np.float64), T[k]) for k in range(len(S))], None,
                              1.0, 1.0, 2, True)
    assert got32.dtype == np.float32
    np.testing.assert_allclose(got32, ref32, rtol=1e-5, atol=0)
    assert np.array_equal(got32, got32.T)


def test_wide_long_pairs_vs_oracle_fp32_and_device_list(twb, oracle):
    """Multi-stripe sweeps with d = 7 and 33 (shared-memory rows, and rows
    too large for shared memory -> per-warp global blocks), fp64 exact,
    fp32 mode, and the ring split over several kernels."""
    rng = np.random.default_rng(77)
    for na, nb, d in [(5000, 4100, 7), (1500, 1700, 33), (700, 900, 200)]:
        va = np.cumsum(rng.standard_normal((na, d)), axis=0)
        vb = np.cumsum(rng.standard_normal((nb, d)), axis=0)
        ta = np.cumsum(rng.uniform(0.1, 1.5, na))
        tb = np.cumsum(rng.uniform(0.1, 1.5, nb))
        want = oracle.twed_tiled(va, ta, vb, tb, 1.0, 1.0, 2, threads=8)
        assert twb.twed(va, ta, vb, tb, 1.0, 1.0, 2) == want, (na, nb, d)
        assert twb.twed(va, ta, vb, tb, 1.0, 1.0, 2, device=[0, 0]) == want, (na, nb, d)
        a32, b32 = va.astype(np.float32), vb.astype(np.float32)
        t32a, t32b = ta.astype(np.float32), tb.astype(np.float32)
        w32 = oracle.twed_tiled(a32.astype(np.float64), t32a.astype(np.float64),
                                b32.astype(np.float64), t32b.astype(np.float64), 1.0, 1.0, 2,
                                threads=8)
        got32 = twb.twed(a32, t32a, b32, t32b, 1.0, 1.0, 2, dtype=np.float32)
        assert got32 == pytest.approx(w32, rel=1e-5), (na, nb, d)


def test_wide_seam_and_prepare(twb, oracle):
    """The S2 seam (band solve on prepared arrays) and the device precompute at d = 9."""
    rng = np.random.default_rng(5)
    va, vb = rng.standard_normal((300, 9)), rng.standard_normal((410, 9))
    ta, tb = np.cumsum(rng.uniform(0.1, 1, 300)), np.cumsum(rng.uniform(0.1, 1, 410))
    params = twb.TwedParams(nu=0.5, lam=0.25, degree=2)
    pa = twb.prepare_series(twb.TimeSeries(va, ta), params)
    pb = twb.prepare_series(twb.TimeSeries(vb, tb), params)
    for got, want in zip(pa, oracle.prepare_series(va, ta, 0.5, 0.25, 2)):
        assert np.array_equal(got, want)
    want = oracle.twed(va, ta, vb, tb, 0.5, 0.25, 2)
    assert twb.band_solve(pa, pb, 0.5, 2) == want


def test_wide_device_resident_ragged_vs_oracle(twb, oracle):
    import torch
    rng = np.random.default_rng(8)
    lens = [1, 5, 64, 129, 300]
    d = 6
    series = [(rng.standard_normal((n, d)), np.cumsum(rng.uniform(0.1, 1, n))) for n in lens]
    want = oracle.twed_batch(series, None, 1.0, 0.5, 2, True)
    AA = torch.tensor(np.concatenate([v for v, _ in series]), device="cuda")
    TA = torch.tensor(np.concatenate([t for _, t in series]), device="cuda")
    off = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    got = twb.twed_batch_dev(AA, off, TA, nu=1.0, lam=0.5, degree=2, tri=True)
    torch.cuda.synchronize()
    assert np.array_equal(got.cpu().numpy(), want)


def test_runtime_d_kernels_on_the_small_goldens():
    """TWB_FORCE_DYN=1 routes every dimension (1..5 here) through the
    runtime-d kernels: they must reproduce all of the reference's small
    goldens (pairs and batches) bit for bit, like the compile-time ones."""
    code = r"""
import sys, json, numpy as np
sys.path[:0] = [{repo!r}, {tests!r}]
from conftest import as_values, dec, same_float
import paper_2007_16135_b200 as twb
from paper_2007_16135_b200 import warpband
g = json.load(open({small!r}))
bad = []
for c in g["pairs"]:
    va = as_values(c["values_a"])
    got = twb.twed(va, as_values(c["times_a"]), as_values(c["values_b"]), as_values(c["times_b"]),
                   nu=c["nu"], lam=c["lam"], degree=c["degree"])
    want = float(dec(c["value"]))
    d = 1 if va.ndim == 1 else va.shape[1]
    ok = same_float(got, want) if (c["degree"] <= 2 or d == 1) else abs(got - want) <= 1e-12 * abs(want)
    if not ok: bad.append((c["name"], got, want))
for c in g["batches"]:
    ser = lambda l: [(as_values(s["values"]), as_values(s["times"])) for s in l]
    la = ser(c["series_a"]); lb = None if c["series_b"] is None else ser(c["series_b"])
    m = warpband.twed_batch(la, lb, nu=c["nu"], lam=c["lam"], degree=c["degree"], symmetric=c["symmetric"])
    if not np.array_equal(m, np.asarray(dec(c["matrix"]))): bad.append(c["name"])
print(json.dumps({{"n": len(g["pairs"]) + len(g["batches"]), "bad": bad}}))
""".format(repo=str(REPO), tests=str(REPO / "tests"), small=str(GOLDEN / "small.json"))
    env = dict(os.environ, TWB_FORCE_DYN="1")
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                         timeout=600)
    assert out.returncode == 0, out.stderr[-3000:]
    res = json.loads(out.stdout.strip().splitlines()[-1])
    assert res["n"] > 250 and res["bad"] == [], res["bad"][:10]
