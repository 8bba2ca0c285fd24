"""GPU property and robustness tests (reference test strategy):
exact symmetry and identity, metric axioms, lambda monotonicity, NaN/inf
inputs on the long-pair kernel, the runtime-degree path, ragged batches,
re-entrancy from many host threads, the S2 seam adapter and the sharded
batch building blocks. Everything calls through the C ABI."""

import math
import threading

import numpy as np
import pytest

from conftest import has_cuda, same_float

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not has_cuda(), reason="needs a CUDA device")]


@pytest.fixture(scope="module")
def twb():
    import paper_2007_16135_b200 as twb
    return twb


def _series(rng, n, d, irregular=True):
    v = np.cumsum(rng.standard_normal((n, d)), axis=0)
    t = np.cumsum(rng.uniform(0.05, 2.0, n)) + rng.uniform(-3, 3) if irregular \
        else np.arange(n, dtype=float)
    return v, t


def test_symmetry_and_identity_exact(twb):
    """test_reference.py:18-21,41-46: twed(a, b) == twed(b, a) bit for bit; twed(a, a) == 0."""
    rng = np.random.default_rng(31)
    for na, nb, d in [(5, 900, 1), (1300, 40, 2), (3000, 2999, 3), (700, 2500, 4)]:
        a, ta = _series(rng, na, d)
        b, tb = _series(rng, nb, d)
        ab = twb.twed(a, ta, b, tb, nu=0.5, lam=0.25, degree=2)
        ba = twb.twed(b, tb, a, ta, nu=0.5, lam=0.25, degree=2)
        assert ab == ba, (na, nb, d)
        assert twb.twed(a, ta, a, ta, nu=0.5, lam=0.25, degree=2) == 0.0


def test_metric_axioms(twb):
    """test_reference.py:65-74 / test_acceptance.py:148-170: triangle inequality
    (1e-9 slack), positivity, lambda monotonicity."""
    rng = np.random.default_rng(32)
    xs = [_series(rng, int(n), 2) for n in rng.integers(300, 1200, size=6)]
    for nu, lam in ((0.1, 0.0), (1.0, 1.0)):
        D = np.array([[twb.twed(x[0], x[1], y[0], y[1], nu=nu, lam=lam, degree=2) for y in xs]
                      for x in xs])
        assert np.all(np.diag(D) == 0.0) and np.all(D[~np.eye(len(xs), dtype=bool)] > 0)
        for i in range(len(xs)):
            for j in range(len(xs)):
                for k in range(len(xs)):
                    assert D[i, k] <= D[i, j] + D[j, k] + 1e-9 * max(1.0, D[i, k])
    a, ta = xs[0]
    b, tb = xs[1]
    vals = [twb.twed(a, ta, b, tb, nu=0.3, lam=lam, degree=2) for lam in (0.0, 0.5, 1.0, 2.0)]
    assert all(x <= y for x, y in zip(vals, vals[1:]))


@pytest.mark.parametrize("bad", ["nan", "inf", "huge", "tiny"])
def test_non_finite_and_extreme_values_long_pair(twb, oracle, bad):
    """The reference rejects non-finite timestamps only (core.py:58-59): NaN and
    inf values flow through its `<` chain. Long pairs (wave kernel) must agree
    bit for bit in the NaN-exact mode."""
    rng = np.random.default_rng(33)
    a, ta = _series(rng, 1500, 2)
    b, tb = _series(rng, 1100, 2)
    val = {"nan": np.nan, "inf": np.inf, "huge": 1e300, "tiny": 1e-200}[bad]
    a[700, 1] = val
    if bad in ("huge", "tiny"):
        b[[3, 900], 0] = val
    got = twb.twed(a, ta, b, tb, nu=1.0, lam=0.5, degree=2)
    want = oracle.twed(a, ta, b, tb, 1.0, 0.5, 2)
    assert same_float(got, want), (bad, got, want)


@pytest.mark.parametrize("degree", [1, 3, 4])
def test_other_degrees_long_pairs(twb, oracle, degree):
    """degree 1 is bit-exact; degree >= 3 with d >= 2 within 1e-12 (libm pow)."""
    rng = np.random.default_rng(34)
    a, ta = _series(rng, 2100, 3)
    b, tb = _series(rng, 1700, 3)
    got = twb.twed(a, ta, b, tb, nu=0.7, lam=0.1, degree=degree)
    want = oracle.twed(a, ta, b, tb, 0.7, 0.1, degree)
    if degree == 1:
        assert got == want
    else:
        assert got == pytest.approx(want, rel=1e-12)


def test_ragged_batch_vs_oracle(twb, oracle):
    rng = np.random.default_rng(35)
    la = [_series(rng, int(n), 2) for n in rng.integers(1, 300, size=41)]
    lb = [_series(rng, int(n), 2) for n in rng.integers(1, 260, size=29)]
    R = twb.twed_batch([x[0] for x in la], [x[1] for x in la], [y[0] for y in lb],
                       [y[1] for y in lb], 0.8, 0.3, 2, False)
    for i in rng.integers(0, len(la), size=25):
        for j in rng.integers(0, len(lb), size=3):
            want = oracle.twed(la[i][0], la[i][1], lb[j][0], lb[j][1], 0.8, 0.3, 2)
            assert R[i, j] == want, (i, j)
    R32 = twb.twed_batch([x[0] for x in la], [x[1] for x in la], [y[0] for y in lb],
                         [y[1] for y in lb], 0.8, 0.3, 2, False, dtype=np.float32)
    for i in rng.integers(0, len(la), size=10):
        j = int(rng.integers(0, len(lb)))
        a32, b32 = (x.astype(np.float32).astype(np.float64) for x in (la[i][0], lb[j][0]))
        ta32, tb32 = (x.astype(np.float32).astype(np.float64) for x in (la[i][1], lb[j][1]))
        want = oracle.twed(a32, ta32, b32, tb32, 0.8, 0.3, 2)
        assert float(R32[i, j]) == pytest.approx(want, rel=1e-5)


def test_many_host_threads(twb, oracle):
    """The C ABI is re-entrant (per-thread stream, per-call scratch); ctypes
    releases the GIL like numba's nogil kernels."""
    rng = np.random.default_rng(36)
    pairs = [(_series(rng, int(rng.integers(200, 3000)), 2),
              _series(rng, int(rng.integers(200, 3000)), 2)) for _ in range(12)]
    want = [oracle.twed(a[0], a[1], b[0], b[1], 1.0, 1.0, 2) for a, b in pairs]
    got = [None] * len(pairs)

    def work(k):
        for _ in range(3):
            a, b = pairs[k]
            got[k] = twb.twed(a[0], a[1], b[0], b[1], nu=1.0, lam=1.0, degree=2)

    threads = [threading.Thread(target=work, args=(k,)) for k in range(len(pairs))]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert got == want


def test_seam_adapter_installs_into_a_reference_like_module(twb, oracle):
    """paper_2007_16135_b200.seam.install swaps _kernels.twed_band_serial /
    _parallel (the S2 seam, _kernels.py:128,146) and restores them."""
    import types

    from paper_2007_16135_b200 import seam

    def cpu_band(*args):
        raise AssertionError("CPU band called")

    kernels = types.SimpleNamespace(twed_band_serial=cpu_band, twed_band_parallel=cpu_band)
    fake = types.SimpleNamespace(_kernels=kernels)
    h = seam.install(fake)
    rng = np.random.default_rng(37)
    a, ta = _series(rng, 800, 3)
    b, tb = _series(rng, 650, 3)
    pa = oracle.prepare_series(a, ta, 0.5, 0.2, 2)
    pb = oracle.prepare_series(b, tb, 0.5, 0.2, 2)
    z = np.zeros(1)
    got = fake._kernels.twed_band_parallel(z, z, z, pa[0], pa[1], pa[2], pb[0], pb[1], pb[2],
                                           0.5, 2)
    assert got == oracle.band_serial(pa, pb, 0.5, 2)
    assert h.calls == 1
    h.restore()
    assert fake._kernels.twed_band_serial is cpu_band


def test_sharded_rows_and_device_mirror(twb):
    """The multi-GPU building blocks on one device: row blocks of a tri batch
    (row_begin/row_end) + on-device mirror == the full symmetric matrix."""
    import torch

    from paper_2007_16135_b200.distributed import row_bounds
    rng = np.random.default_rng(38)
    N, n, d = 97, 64, 2
    S = np.cumsum(rng.standard_normal((N, n, d)), axis=1)
    T = np.broadcast_to(np.arange(n, dtype=float), (N, n)).copy()
    full = twb.twed_batch(S, T, None, None, 1.0, 0.5, 2, True)
    dev = torch.device("cuda:0")
    dS = torch.from_numpy(S.reshape(-1, d)).to(dev)
    dT = torch.from_numpy(T.reshape(-1)).to(dev)
    off = np.arange(N + 1, dtype=np.int64) * n
    M = torch.zeros((N, N), dtype=torch.float64, device=dev)
    for b0, b1 in row_bounds(N, 3, True):
        blk = twb.twed_batch_dev(dS, off, dT, nu=1.0, lamb=0.5, degree=2, tri=True,
                                 row_begin=b0, row_end=b1)
        M[b0:b1] = blk
    twb.mirror_upper_dev(M)
    torch.cuda.synchronize()
    assert np.array_equal(M.cpu().numpy(), full)


def test_single_sample_and_tiny_series(twb, oracle):
    """Edge sizes (test_core.py / test_band.py): n = 1 against long, 1 x 1."""
    rng = np.random.default_rng(39)
    for na, nb in [(1, 1), (1, 5000), (4000, 1), (2, 3)]:
        a, ta = _series(rng, na, 3)
        b, tb = _series(rng, nb, 3)
        got = twb.twed(a, ta, b, tb, nu=1.0, lam=1.0, degree=2)
        assert got == oracle.twed(a, ta, b, tb, 1.0, 1.0, 2), (na, nb)
    assert math.isfinite(got)


def test_reference_cli_on_the_gpu_backend(tmp_path, small_golden):
    """paper_2007_16135_b200.refcli: the reference's own CLI (cli.py:95-115) with
    the band on libtwb200 reproduces its frozen fixture distance
    (test_cli.py:25-27, 38.32093438282728). Needs the reference package
    (baseline/_ref, staged by scripts/stage_reference.sh)."""
    import contextlib
    import io
    import os
    import sys
    from pathlib import Path

    ref = Path(__file__).resolve().parents[1] / "baseline" / "_ref"
    if not (ref / "twedband").is_dir():
        pytest.skip("reference package not staged in baseline/_ref")
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/twb_numba_cache")
    sys.path.insert(0, str(ref))
    try:
        import twedband  # noqa: F401
    except Exception as exc:  # numba missing
        pytest.skip(f"reference package not importable: {exc}")
    from conftest import as_values
    from paper_2007_16135_b200 import refcli
    case = small_golden["pairs"][0]
    assert case["name"] == "fixture_pair_nu1_lam0"
    for name, vk, tk in (("a", "values_a", "times_a"), ("b", "values_b", "times_b")):
        v, t = as_values(case[vk]), as_values(case[tk])
        v = v.reshape(len(t), -1)
        lines = ["t," + ",".join(f"v{k}" for k in range(v.shape[1]))]
        lines += [",".join([repr(float(t[i]))] + [repr(float(x)) for x in v[i]])
                  for i in range(len(t))]
        (tmp_path / f"{name}.csv").write_text("\n".join(lines) + "\n")
    buf = io.StringIO()
    with contextlib.redirect_stdout(buf):
        rc = refcli.main(["twed", str(tmp_path / "a.csv"), str(tmp_path / "b.csv")])
    assert rc == 0
    assert "38.32093438282728" in buf.getvalue(), buf.getvalue()
