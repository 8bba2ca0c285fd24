"""One pair over several devices (twb_twed_multi_*).

The run has one B200, so the ring of CTAs is split over several kernels on
that one device (``device=[0, 0]``): each kernel is its own cooperative launch
on its own stream, the last CTA of each part feeds the next part's CTA 0
through its inbox with system-scope release/acquire, exactly the protocol of
the multi-GPU case minus the NVLink hop. Results must be bit-identical to the
single-kernel sweep and to the reference goldens.
"""

import os

import numpy as np
import pytest

from conftest import has_cuda

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not has_cuda(), reason="needs a CUDA device")]

os.environ.setdefault("TWB_RING_TIMEOUT_MS", "15000")


@pytest.fixture(scope="module")
def twb():
    import paper_2007_16135_b200 as twb
    return twb


@pytest.mark.parametrize("parts", [[0, 0], [0, 0, 0], [0, 0, 0, 0]])
def test_ring_parts_match_single_kernel(twb, config_golden, parts):
    from paper_2007_16135_b200.workloads import make_pair
    g = config_golden["cfg2"]  # n = 100k, d = 1 (the reference's own value)
    a, ta, b, tb = make_pair(100_000, 1, 1)
    assert twb.twed(a, ta, b, tb, 1.0, 1.0, 2, device=parts) == g["value"]
    for key in ("walk_8192_d3_s13", "walk_20000_d1_s14"):
        g = config_golden[key]
        a, ta, b, tb = make_pair(g["n"], g["d"], g["seed"])
        assert twb.twed(a, ta, b, tb, 1.0, 1.0, 2, device=parts) == g["value"], key


def test_ring_long_pair_d3(twb):
    """Several rounds of stripes over the ring (n = 400k, d = 3)."""
    from paper_2007_16135_b200.workloads import make_pair
    a, ta, b, tb = make_pair(400_000, 3, 21)
    one = twb.twed(a, ta, b, tb, 1.0, 1.0, 2)
    assert twb.twed(a, ta, b, tb, 1.0, 1.0, 2, device=[0, 0]) == one
    assert twb.twed(a, ta, b, tb, 1.0, 1.0, 2, device=[0, 0, 0]) == one


def test_ring_ragged_irregular_fp32_and_nan(twb):
    rng = np.random.default_rng(5)
    a = np.cumsum(rng.standard_normal((37_001, 2)), axis=0)
    b = np.cumsum(rng.standard_normal((52_333, 2)), axis=0)
    ta = np.cumsum(rng.uniform(0.05, 2.0, len(a)))
    tb = np.cumsum(rng.uniform(0.05, 2.0, len(b)))
    for nu, lam in ((1.0, 1.0), (0.25, 0.5)):
        one = twb.twed(a, ta, b, tb, nu, lam, 2)
        assert twb.twed(a, ta, b, tb, nu, lam, 2, device=[0, 0]) == one
    one = twb.twed(a, ta, b, tb, 1.0, 1.0, 2, dtype=np.float32)
    assert twb.twed(a, ta, b, tb, 1.0, 1.0, 2, dtype=np.float32, device=[0, 0]) == one
    a2 = a.copy()
    a2[20_000, 1] = np.nan  # NaN-exact mode (compare chain, no swap)
    one = twb.twed(a2, ta, b, tb, 1.0, 1.0, 2)
    got = twb.twed(a2, ta, b, tb, 1.0, 1.0, 2, device=[0, 0])
    assert (np.isnan(one) and np.isnan(got)) or got == one


def test_ring_bad_device_raises(twb):
    a = np.arange(100.0)
    with pytest.raises(ValueError, match="out of range"):
        twb.twed(a, a, a, a, 1.0, 1.0, 2, device=[0, 99])


@pytest.mark.parametrize("na,nb", [(1, 1), (1, 7), (5, 3), (40, 1000), (1000, 40), (3000, 2999)])
def test_ring_tiny_and_skewed_shapes(twb, na, nb):
    """Fewer stripes than kernels (parts left without a CTA drop out of the ring)."""
    rng = np.random.default_rng(na * 1000 + nb)
    a = np.cumsum(rng.standard_normal((na, 2)), axis=0)
    b = np.cumsum(rng.standard_normal((nb, 2)), axis=0)
    ta, tb = np.arange(na, dtype=float), np.arange(nb, dtype=float)
    one = twb.twed(a, ta, b, tb, 1.0, 1.0, 2)
    assert twb.twed(a, ta, b, tb, 1.0, 1.0, 2, device=[0, 0, 0]) == one


@pytest.mark.parametrize("tri", [False, True])
def test_batch_over_device_list(twb, tri):
    """twed_batch(..., device=[...]): row blocks on several devices (here the one
    B200 twice), one host thread each; identical to the single-device matrix."""
    rng = np.random.default_rng(7)
    series = [np.cumsum(rng.standard_normal((int(n), 2)), axis=0)
              for n in rng.integers(5, 300, 57)]
    one = twb.twed_batch(series, None, None, None, 1.0, 1.0, 2, tri)
    two = twb.twed_batch(series, None, None, None, 1.0, 1.0, 2, tri, device=[0, 0, 0])
    assert np.array_equal(one, two)
    if not tri:
        other = [np.cumsum(rng.standard_normal((64, 2)), axis=0) for _ in range(9)]
        one = twb.twed_batch(series, None, other, None, 1.0, 1.0, 2)
        two = twb.twed_batch(series, None, other, None, 1.0, 1.0, 2, device=[0, 0])
        assert np.array_equal(one, two)


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_batch_multi_abi_triangle_written_on_device(twb, dtype):
    """twb_twed_batch_multi_*: 4 row blocks of a 700-series ragged triangle;
    each block writes its rows and the transposed mirror strip of its upper
    part from the device (no host mirror pass). Equal to one device, and
    exactly symmetric with a zero diagonal."""
    rng = np.random.default_rng(71)
    series = [np.cumsum(rng.standard_normal((int(n), 3)), axis=0)
              for n in rng.integers(1, 260, 700)]
    one = twb.twed_batch(series, None, None, None, 1.0, 0.5, 2, True, dtype=dtype)
    four = twb.twed_batch(series, None, None, None, 1.0, 0.5, 2, True, dtype=dtype,
                          device=[0, 0, 0, 0])
    assert four.dtype == dtype
    assert np.array_equal(one, four)
    assert np.array_equal(four, four.T) and np.all(np.diag(four) == 0)


@pytest.mark.parametrize("degree,d", [(1, 3), (3, 2), (2, 1), (2, 4)])
def test_ring_other_degrees_and_dims(twb, degree, d):
    """Degree 1 (sums of |diff|), degree 3 (the NaN-exact compare chain with a
    runtime degree), d = 1 and d = 4 through the multi-kernel ring."""
    rng = np.random.default_rng(degree * 10 + d)
    a = np.cumsum(rng.standard_normal((12_000, d)), axis=0)
    b = np.cumsum(rng.standard_normal((9_000, d)), axis=0)
    ta, tb = np.arange(len(a), dtype=float), np.arange(len(b), dtype=float)
    one = twb.twed(a, ta, b, tb, 0.5, 0.25, degree)
    assert twb.twed(a, ta, b, tb, 0.5, 0.25, degree, device=[0, 0]) == one


@pytest.mark.parametrize("tri", [False, True])
def test_batch_long_rows_on_stream_pool(twb, tri):
    """Row-side series longer than the warp kernel's 256 samples go through
    per-pair wavefront sweeps spread over a pool of streams: entries equal the
    single-pair results, the triangle layout included."""
    rng = np.random.default_rng(11)
    lens = [200, 257, 300, 511, 900, 64, 1500, 256, 700, 333, 40]
    series = [np.cumsum(rng.standard_normal((n, 2)), axis=0) for n in lens]
    R = twb.twed_batch(series, None, None, None, 1.0, 1.0, 2, tri)
    for i in range(len(series)):
        for j in range(len(series)):
            want = twb.twed(series[i], np.arange(lens[i], dtype=float), series[j],
                            np.arange(lens[j], dtype=float), 1.0, 1.0, 2)
            assert R[i, j] == want, (i, j)
