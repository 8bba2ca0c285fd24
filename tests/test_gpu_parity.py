"""GPU parity: the sm_100a kernels (through the C ABI) vs the reference's goldens
and the pinned CPU oracle.

Bar (BASELINE.json north_star): fp64 bit-identical to the reference (degree 1
and 2, any d; degree >= 3 with d >= 2 within 1e-12 relative: libm pow vs CUDA
pow decide the last bits); fp32 mode within 1e-5 relative of the fp64
reference on the fp32-rounded inputs; batch index and triangle layout exact.
"""

import json
import math

import numpy as np
import pytest

from conftest import GOLDEN, as_values, dec, has_cuda, same_float

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not has_cuda(), reason="needs a CUDA device")]

FP32_RTOL = 1e-5
DEG3_RTOL = 1e-12


@pytest.fixture(scope="module")
def twb():
    import paper_2007_16135_b200 as twb
    return twb


def _exact_expected(case):
    va = np.asarray(dec(case["values_a"]))
    return case["degree"] <= 2 or va.ndim == 1 or va.shape[1] == 1


def test_library_loaded_is_in_tree(twb):
    from paper_2007_16135_b200 import _lib
    lib = _lib.load()
    assert str(_lib.LIB_PATH) == lib._name
    assert _lib.device_count() >= 1


def test_small_pairs_bit_exact(twb, small_golden):
    for case in small_golden["pairs"]:
        got = twb.twed(as_values(case["values_a"]), as_values(case["times_a"]),
                       as_values(case["values_b"]), as_values(case["times_b"]),
                       nu=case["nu"], lam=case["lam"], degree=case["degree"])
        want = float(dec(case["value"]))
        if _exact_expected(case):
            assert same_float(got, want), (case["name"], got, want)
        else:
            assert got == pytest.approx(want, rel=DEG3_RTOL), case["name"]


def test_north_star_spelling(twb, small_golden):
    case = small_golden["pairs"][1]  # readme sin pair, nu=0.1, lam=0.5
    args = [as_values(case[k]) for k in ("values_a", "times_a", "values_b", "times_b")]
    got = twb.twed(*args, case["nu"], case["lam"], case["degree"])
    assert got == float(case["value"]) == 23.953161165093555
    assert twb.twed(*args, nu=case["nu"], lamb=case["lam"], degree=2) == got


def _series(lst):
    return [(as_values(s["values"]), as_values(s["times"])) for s in lst]


def test_batches_bit_exact(twb, small_golden):
    from paper_2007_16135_b200 import warpband
    for case in small_golden["batches"]:
        la = _series(case["series_a"])
        lb = None if case["series_b"] is None else _series(case["series_b"])
        want = np.asarray(dec(case["matrix"]))
        got = warpband.twed_batch(la, lb, nu=case["nu"], lam=case["lam"], degree=case["degree"],
                                  symmetric=case["symmetric"])
        assert got.shape == want.shape
        assert np.array_equal(got, want), case["name"]
        got2 = twb.twed_batch([v for v, _ in la], [t for _, t in la],
                              None if lb is None else [v for v, _ in lb],
                              None if lb is None else [t for _, t in lb],
                              case["nu"], case["lam"], case["degree"], case["symmetric"])
        assert np.array_equal(got2, want), case["name"]


def test_random_pairs_vs_oracle(twb, oracle):
    rng = np.random.default_rng(123)
    for k in range(60):
        na, nb = (int(x) for x in rng.integers(1, 700, size=2))
        if k % 10 == 0:
            na = int(rng.integers(2000, 6000))
        d = int(rng.integers(1, 5))
        deg = int(rng.integers(1, 3))
        nu, lam = float(rng.choice([0.0, 0.1, 1.0, 2.5])), float(rng.choice([0.0, 0.5, 1.0]))
        va, vb = rng.standard_normal((na, d)) * 3, rng.standard_normal((nb, d)) * 3
        ta = np.cumsum(rng.uniform(0.05, 2.0, na)) + rng.uniform(-5, 5)
        tb = np.cumsum(rng.uniform(0.05, 2.0, nb)) + rng.uniform(-5, 5)
        got = twb.twed(va, ta, vb, tb, nu=nu, lam=lam, degree=deg)
        want = oracle.twed_tiled(va, ta, vb, tb, nu, lam, deg, threads=4)
        assert got == want, (k, na, nb, d, deg, nu, lam, got, want)


def test_config_goldens_fp64(twb, config_golden):
    from paper_2007_16135_b200.workloads import make_pair
    a, ta, b, tb = make_pair(1000, 1, 0)
    assert twb.twed(a, ta, b, tb, 1.0, 1.0, 2) == config_golden["cfg1"]["value"]
    for key in ("walk_4096_d1_s11", "walk_3000_d3_s12", "walk_8192_d3_s13", "walk_20000_d1_s14"):
        g = config_golden[key]
        a, ta, b, tb = make_pair(g["n"], g["d"], g["seed"])
        assert twb.twed(a, ta, b, tb, 1.0, 1.0, 2) == g["value"], key
        # symmetry is exact (reference test_reference.py:41-46)
        assert twb.twed(b, tb, a, ta, 1.0, 1.0, 2) == g["value"], key


def test_cfg2_100k_golden(twb, config_golden):
    from paper_2007_16135_b200.workloads import make_pair
    a, ta, b, tb = make_pair(100_000, 1, 1)
    assert twb.twed(a, ta, b, tb, 1.0, 1.0, 2) == config_golden["cfg2"]["value"]


def test_fp32_mode_pairs(twb, config_golden):
    from paper_2007_16135_b200.workloads import make_pair
    a, ta, b, tb = make_pair(1000, 1, 0)
    got = twb.twed(a, ta, b, tb, 1.0, 1.0, 2, dtype=np.float32)
    assert got == pytest.approx(config_golden["cfg1_f32in"]["value"], rel=FP32_RTOL)
    for key in ("walk_3000_d3_s12", "walk_8192_d3_s13", "walk_20000_d1_s14"):
        g = config_golden[key]
        a, ta, b, tb = make_pair(g["n"], g["d"], g["seed"])
        got = twb.twed(a, ta, b, tb, 1.0, 1.0, 2, dtype=np.float32)
        assert got == pytest.approx(config_golden[key + "_f32in"]["value"], rel=FP32_RTOL), key


def test_cfg3_1m_pair(twb):
    """n = 1,000,000, d = 3 (BASELINE cfg3): fp64 vs the oracle golden when it
    exists; always the size-independent properties (fp32 within 1e-5 of fp64,
    identity = 0)."""
    from paper_2007_16135_b200.workloads import make_pair
    a, ta, b, tb = make_pair(1_000_000, 3, 2)
    v64 = twb.twed(a, ta, b, tb, 1.0, 1.0, 2)
    v32 = twb.twed(a, ta, b, tb, 1.0, 1.0, 2, dtype=np.float32)
    path = GOLDEN / "cfg3.json"
    g = json.loads(path.read_text()) if path.exists() else {}
    if "cfg3_n1000000" in g:
        assert v64 == g["cfg3_n1000000"]["value"]
    if "cfg3_n1000000_f32in" in g:
        assert v32 == pytest.approx(g["cfg3_n1000000_f32in"]["value"], rel=FP32_RTOL)
    assert v32 == pytest.approx(v64, rel=FP32_RTOL)
    assert math.isfinite(v64) and v64 > 0


def test_cfg3_64k_golden(twb):
    from paper_2007_16135_b200.workloads import make_pair
    g = json.loads((GOLDEN / "cfg3.json").read_text())
    a, ta, b, tb = make_pair(65536, 3, 2)
    assert twb.twed(a, ta, b, tb, 1.0, 1.0, 2) == g["cfg3_n65536"]["value"]
    got = twb.twed(a, ta, b, tb, 1.0, 1.0, 2, dtype=np.float32)
    assert got == pytest.approx(g["cfg3_n65536_f32in"]["value"], rel=FP32_RTOL)


def test_cfg4_full_batch(twb, config_golden, oracle):
    from paper_2007_16135_b200.workloads import make_set
    AA, TAA = make_set(1000, 256, 1, 3)
    BB, TBB = make_set(1000, 256, 1, 4)
    R = twb.twed_batch(AA, TAA, BB, TBB, 1.0, 1.0, 2, False)
    assert R.shape == (1000, 1000) and R.dtype == np.float64
    for key, want in config_golden["cfg4"]["entries"].items():
        i, j = map(int, key.split(","))
        assert R[i, j] == want, key
    rng = np.random.default_rng(5)
    for i, j in rng.integers(0, 1000, size=(40, 2)):
        assert R[i, j] == oracle.twed(AA[i], TAA[i], BB[j], TBB[j], 1.0, 1.0, 2), (i, j)


def test_cfg5_tri_fp32(twb, config_golden, oracle):
    from paper_2007_16135_b200.workloads import make_set
    S, TS = make_set(10000, 128, 2, 5)
    R = twb.twed_batch(S, TS, None, None, 1.0, 1.0, 2, True, dtype=np.float32)
    assert R.shape == (10000, 10000) and R.dtype == np.float32
    assert np.array_equal(R, R.T)
    assert np.all(np.diag(R) == 0.0)
    S64 = S.astype(np.float32).astype(np.float64)
    for key, want in config_golden["cfg5_f32in"]["entries"].items():
        i, j = map(int, key.split(","))
        assert R[i, j] == pytest.approx(want, rel=FP32_RTOL, abs=0.0), key
    rng = np.random.default_rng(6)
    for i, j in rng.integers(0, 10000, size=(30, 2)):
        want = oracle.twed(S64[i], TS[i], S64[j], TS[j], 1.0, 1.0, 2)
        assert float(R[i, j]) == pytest.approx(want, rel=FP32_RTOL), (i, j)


def test_tri_equals_full(twb):
    rng = np.random.default_rng(8)
    series = [rng.standard_normal((int(n), 2)) for n in rng.integers(1, 300, size=37)]
    full = twb.twed_batch(series, None, None, None, 0.5, 0.25, 2, False)
    tri = twb.twed_batch(series, None, None, None, 0.5, 0.25, 2, True)
    assert np.array_equal(full, tri)
    assert np.array_equal(tri, tri.T)


def test_batch_long_rows_fall_back_to_wavefront(twb, oracle):
    rng = np.random.default_rng(9)
    la = [rng.standard_normal((n, 1)) for n in (300, 20, 700)]
    lb = [rng.standard_normal((n, 1)) for n in (5, 400)]
    R = twb.twed_batch(la, None, lb, None, 1.0, 0.5, 2)
    for i, a in enumerate(la):
        for j, b in enumerate(lb):
            want = oracle.twed(a, np.arange(len(a), dtype=float), b,
                               np.arange(len(b), dtype=float), 1.0, 0.5, 2)
            assert R[i, j] == want


def test_band_solve_seam(twb, oracle, small_golden):
    for case in small_golden["pairs"][:40]:
        pa = oracle.prepare_series(as_values(case["values_a"]), as_values(case["times_a"]),
                                   case["nu"], case["lam"], case["degree"])
        pb = oracle.prepare_series(as_values(case["values_b"]), as_values(case["times_b"]),
                                   case["nu"], case["lam"], case["degree"])
        got = twb.band_solve(pa, pb, case["nu"], case["degree"])
        want = oracle.band_serial(pa, pb, case["nu"], case["degree"])
        if _exact_expected(case):
            assert same_float(got, want), case["name"]
        else:
            assert got == pytest.approx(want, rel=DEG3_RTOL)


def test_prepare_series_device(twb, oracle, small_golden):
    from paper_2007_16135_b200 import TimeSeries, TwedParams
    for case in small_golden["pairs"][4:30]:
        s = TimeSeries(as_values(case["values_a"]), as_values(case["times_a"]))
        p = TwedParams(case["nu"], case["lam"], case["degree"])
        got = twb.prepare_series(s, p)
        want = oracle.prepare_series(s.values, s.timestamps, p.nu, p.lam, p.degree)
        for x, y in zip(got, want):
            if case["degree"] <= 2 or s.d == 1:
                assert np.array_equal(x, y)
            else:
                np.testing.assert_allclose(x, y, rtol=1e-13)


def test_device_resident_api(twb):
    import torch
    from paper_2007_16135_b200.workloads import make_pair
    a, ta, b, tb = make_pair(5000, 2, 21)
    want = twb.twed(a, ta, b, tb, 1.0, 1.0, 2)
    dev = torch.device("cuda:0")
    t = [torch.from_numpy(np.ascontiguousarray(x)).to(dev) for x in (a, ta, b, tb)]
    out = twb.twed_dev(*t, nu=1.0, lamb=1.0, degree=2)
    torch.cuda.synchronize()
    assert out.item() == want


def test_sqrt_split_bit_exact(twb):
    """The DP kernels' straight-line fp64 sqrt equals __dsqrt_rn bit for bit."""
    import ctypes
    from paper_2007_16135_b200 import _lib
    lib = _lib.load()
    fast = ctypes.c_int64(0)
    bad = lib.twb_selftest_sqrt(1 << 26, 20261017, 0, ctypes.byref(fast))
    assert bad == 0, bad
    assert fast.value > (1 << 24)


@pytest.mark.parametrize("scale", [1e-170, 1e-150, 1.0, 1e150, 1e240])
def test_extreme_magnitudes_vs_oracle(twb, oracle, scale):
    """Tiny and huge values send sqrt arguments outside the fast path (zero,
    denormal squares) or close to overflow; results stay bit-identical."""
    rng = np.random.default_rng(int(abs(np.log10(scale))) + 7)
    for d in (2, 3):
        a = np.cumsum(rng.standard_normal((300, d)), axis=0) * scale
        b = np.cumsum(rng.standard_normal((257, d)), axis=0) * scale
        b[::17] = a[:len(b[::17])]  # exact matches -> zero distances
        ta, tb = np.arange(300.0), np.arange(257.0)
        for nu, lam in ((1.0, 1.0), (0.5, 0.0)):
            got = twb.twed(a, ta, b, tb, nu=nu, lam=lam, degree=2)
            want = oracle.twed(a, ta, b, tb, nu, lam, 2)
            assert same_float(got, want), (scale, d, nu, lam, got, want)
            R = twb.twed_batch([a, b, a[:100]], None, None, None, nu, lam, 2, True)
            assert same_float(R[0, 1], want)
            assert R[0, 0] == 0.0 and R[1, 1] == 0.0


def test_validation_messages(twb):
    with pytest.raises(ValueError, match="3 timestamps for 2 samples"):
        twb.twed([[1.0], [2.0]], [0.0, 1.0, 2.0], [1.0], [0.0])
    with pytest.raises(ValueError, match="3 dimensions"):
        twb.twed(np.zeros((2, 2, 2)), [0.0, 1.0], [1.0], [0.0])
    with pytest.raises(ValueError, match="A has d=2, B has d=1"):
        twb.twed([[1.0, 2.0]], [0.0], [1.0], [0.0])
    with pytest.raises(twb.InvalidInputError, match="strictly increasing"):
        twb.twed([1.0, 2.0], [1.0, 1.0], [1.0], [0.0])
    with pytest.raises(twb.InvalidInputError):
        twb.twed_batch([np.array([1.0])], None, [np.array([2.0])], None, tri=True)


def test_device_api_is_async_and_graph_capturable(twb):
    """twed_dev makes the safe / NaN-exact choice on the device (no host round
    trip), so it can be captured in a CUDA graph and replayed on new data."""
    import torch
    from paper_2007_16135_b200.workloads import make_pair
    dev = torch.device("cuda:0")
    a, ta, b, tb = make_pair(3000, 3, 31)
    t = [torch.from_numpy(np.ascontiguousarray(x)).to(dev) for x in (a, ta, b, tb)]
    out = torch.empty(1, dtype=torch.float64, device=dev)
    twb.twed_dev(*t, nu=1.0, lamb=1.0, degree=2, out=out)  # warm (kernel attributes)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        twb.twed_dev(*t, nu=1.0, lamb=1.0, degree=2, out=out)
    for seed in (32, 33):
        a2, ta2, b2, tb2 = make_pair(3000, 3, seed)
        if seed == 33:
            a2[1234, 1] = np.nan  # the captured graph takes the NaN-exact sweep
        for dst, src in zip(t, (a2, ta2, b2, tb2)):
            dst.copy_(torch.from_numpy(np.ascontiguousarray(src)))
        g.replay()
        torch.cuda.synchronize()
        want = twb.twed(a2, ta2, b2, tb2, 1.0, 1.0, 2)
        got = out.item()
        assert (math.isnan(want) and math.isnan(got)) or got == want, (seed, got, want)
