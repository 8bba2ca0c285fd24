"""GPU parity at full matrix scale and through the device-resident entry points.

- config 4 (1000 x 1000 full, n = 256, d = 1, fp64): EVERY entry equals the
  pinned C oracle (engine.py:183-226 restated, tests/test_oracle_golden.py pins
  it to the reference), bit for bit;
- config 5 (10k x 10k tri, n = 128, d = 2, fp32): the 1000-series leading
  sub-triangle against the oracle on the fp32-rounded inputs within 1e-5
  relative, plus the exact symmetric layout of the whole matrix;
- twed_batch_dev / twed_dev (packed device tensors, CSR offsets, the paper's
  twed_dev) on ragged lengths 1..300 against the oracle -- not
  against this library's own host API.
"""

import math

import numpy as np
import pytest

from conftest import has_cuda, same_float

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not has_cuda(), reason="needs a CUDA device")]

FP32_RTOL = 1e-5


@pytest.fixture(scope="module")
def twb():
    import paper_2007_16135_b200 as twb
    return twb


def _walks(rng, lengths, d, irregular=False):
    out = []
    for n in lengths:
        v = np.cumsum(rng.standard_normal((int(n), d)), axis=0)
        if irregular:  # conftest-style strictly increasing timestamps (T/conftest.py:19-21)
            t = rng.uniform(0.0, 5.0) + np.cumsum(rng.uniform(0.05, 2.0, int(n)))
        else:
            t = np.arange(int(n), dtype=np.float64)
        out.append((v, t))
    return out


def _pack_dev(series, dtype, dev):
    import torch
    vals = np.concatenate([np.asarray(v, dtype=np.float64).reshape(len(t), -1) for v, t in series])
    times = np.concatenate([np.asarray(t, dtype=np.float64) for _, t in series])
    off = np.zeros(len(series) + 1, dtype=np.int64)
    off[1:] = np.cumsum([len(t) for _, t in series])
    return (torch.from_numpy(np.ascontiguousarray(vals.astype(dtype))).to(dev), off,
            torch.from_numpy(np.ascontiguousarray(times.astype(dtype))).to(dev))


def test_cfg4_whole_matrix_equals_oracle(twb, oracle):
    from paper_2007_16135_b200.workloads import make_set
    AA, TAA = make_set(1000, 256, 1, 3)
    BB, TBB = make_set(1000, 256, 1, 4)
    R = twb.twed_batch(AA, TAA, BB, TBB, 1.0, 1.0, 2, False)
    W = oracle.twed_batch([(AA[i], TAA[i]) for i in range(1000)],
                          [(BB[j], TBB[j]) for j in range(1000)], 1.0, 1.0, 2, False, threads=0)
    bad = np.argwhere(R.view(np.int64) != W.view(np.int64))
    assert bad.size == 0, (len(bad), bad[:5])


def test_cfg5_subtriangle_vs_oracle(twb, oracle):
    from paper_2007_16135_b200.workloads import make_set
    S, TS = make_set(10000, 128, 2, 5)
    R = twb.twed_batch(S, TS, None, None, 1.0, 1.0, 2, True, dtype=np.float32)
    assert R.shape == (10000, 10000) and R.dtype == np.float32
    assert np.array_equal(R, R.T) and np.all(np.diag(R) == 0.0)
    m = 1000
    S64 = S[:m].astype(np.float32).astype(np.float64)
    T64 = TS[:m].astype(np.float32).astype(np.float64)
    W = oracle.twed_batch([(S64[k], T64[k]) for k in range(m)], None, 1.0, 1.0, 2, True, threads=0)
    got = R[:m, :m].astype(np.float64)
    iu = np.triu_indices(m, 1)
    rel = np.abs(got[iu] - W[iu]) / np.abs(W[iu])
    assert rel.max() <= FP32_RTOL, (rel.max(), np.unravel_index(np.argmax(rel), rel.shape))
    assert np.all(np.diag(W) == 0.0)


@pytest.mark.parametrize("d", [1, 2, 3, 7])
def test_ragged_batch_dev_vs_oracle(twb, oracle, d):
    import torch
    dev = torch.device("cuda:0")
    rng = np.random.default_rng(100 + d)
    la = _walks(rng, rng.integers(1, 301, size=23), d, irregular=True)
    lb = _walks(rng, rng.integers(1, 301, size=17), d, irregular=True)
    la[0] = (la[0][0][:1], la[0][1][:1])  # a single-sample series
    nu, lam = 0.75, 0.5
    AA, aoff, TAA = _pack_dev(la, np.float64, dev)
    BB, boff, TBB = _pack_dev(lb, np.float64, dev)
    # full, then a row range of the same matrix
    R = twb.twed_batch_dev(AA, aoff, TAA, BB, boff, TBB, nu=nu, lamb=lam, degree=2).cpu().numpy()
    W = oracle.twed_batch(la, lb, nu, lam, 2, False, threads=0)
    assert np.array_equal(R.view(np.int64), W.view(np.int64))
    R2 = twb.twed_batch_dev(AA, aoff, TAA, BB, boff, TBB, nu=nu, lamb=lam, degree=2,
                            row_begin=5, row_end=19).cpu().numpy()
    assert np.array_equal(R2.view(np.int64), W[5:19].view(np.int64))
    # self batch in the tri layout (upper computed, mirrored)
    T = twb.twed_batch_dev(AA, aoff, TAA, nu=nu, lamb=lam, degree=2, tri=True).cpu().numpy()
    WT = oracle.twed_batch(la, None, nu, lam, 2, True, threads=0)
    assert np.array_equal(T.view(np.int64), WT.view(np.int64))
    # fp32 inputs, fp32 matrix: 1e-5 of the fp64 oracle on the rounded inputs
    A32, _, TA32 = _pack_dev(la, np.float32, dev)
    B32, _, TB32 = _pack_dev(lb, np.float32, dev)
    R32 = twb.twed_batch_dev(A32, aoff, TA32, B32, boff, TB32, nu=nu, lamb=lam,
                             degree=2).cpu().numpy()
    r32 = lambda L: [(np.asarray(v, np.float32).astype(np.float64),
                      np.asarray(t, np.float32).astype(np.float64)) for v, t in L]
    W32 = oracle.twed_batch(r32(la), r32(lb), nu, lam, 2, False, threads=0)
    np.testing.assert_allclose(R32.astype(np.float64), W32, rtol=FP32_RTOL, atol=0)


@pytest.mark.parametrize("d", [1, 3, 6])
def test_ragged_twed_dev_vs_oracle(twb, oracle, d):
    import torch
    dev = torch.device("cuda:0")
    rng = np.random.default_rng(200 + d)
    out = torch.empty(1, dtype=torch.float64, device=dev)
    for na, nb in ((1, 1), (1, 777), (300, 1), (257, 4099), (5000, 3001), (2048, 2048)):
        (a, ta), (b, tb) = _walks(rng, (na, nb), d, irregular=True)
        for nu, lam in ((1.0, 1.0), (0.1, 0.0)):
            t = [torch.from_numpy(np.ascontiguousarray(x)).to(dev) for x in (a, ta, b, tb)]
            twb.twed_dev(*t, nu=nu, lamb=lam, degree=2, out=out)
            got = out.item()
            want = oracle.twed(a, ta, b, tb, nu, lam, 2)
            assert same_float(got, want), (na, nb, nu, lam, got, want)
            t32 = [torch.from_numpy(np.ascontiguousarray(x.astype(np.float32))).to(dev)
                   for x in (a, ta, b, tb)]
            twb.twed_dev(*t32, nu=nu, lamb=lam, degree=2, out=out)
            w32 = oracle.twed(*(x.astype(np.float32).astype(np.float64) for x in (a, ta, b, tb)),
                              nu, lam, 2)
            assert out.item() == pytest.approx(w32, rel=FP32_RTOL), (na, nb, nu, lam)


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
@pytest.mark.parametrize("d", [1, 3, 5, 20])
def test_fused_prepare_vs_oracle(twb, oracle, dtype, d):
    """The single pair's precompute (one launch: both series, bulk-copy staged
    tiles, fused input check) equals core.prepare_series (C:218-234) row for
    row, in the DP kernels' layout (virtual row +inf), for every alignment of
    the input pointers (the bulk copies' unaligned heads and tails)."""
    import ctypes
    import torch
    from paper_2007_16135_b200 import _lib
    lib = _lib.load()
    dev = torch.device("cuda:0")
    rng = np.random.default_rng(300 + d)
    f32 = dtype == np.float32
    fn = lib.twb_prepare_pair_dev_f32 if f32 else lib.twb_prepare_pair_dev_f64
    rdt = torch.float32 if f32 else torch.float64
    for na, nb, shift in ((1, 2, 0), (255, 257, 1), (1000, 3001, 2), (70001, 513, 3)):
        a = np.cumsum(rng.standard_normal((na, d)), axis=0).astype(dtype)
        b = np.cumsum(rng.standard_normal((nb, d)), axis=0).astype(dtype)
        ta = np.cumsum(rng.uniform(0.05, 2.0, na)).astype(dtype)
        tb = np.cumsum(rng.uniform(0.05, 2.0, nb)).astype(dtype)

        def shifted(x):  # device copy whose data pointer is `shift` elements past 16-byte alignment
            buf = torch.empty(x.size + 8, dtype=rdt, device=dev)
            v = buf[shift:shift + x.size]
            v.copy_(torch.from_numpy(np.ascontiguousarray(x).reshape(-1)))
            return v
        ins = [shifted(x) for x in (a, ta, b, tb)]
        VA = torch.empty((na + 1) * d, dtype=rdt, device=dev)
        VB = torch.empty((nb + 1) * d, dtype=rdt, device=dev)
        TA_ = torch.empty(na + 1, dtype=rdt, device=dev)
        TB_ = torch.empty(nb + 1, dtype=rdt, device=dev)
        DA = torch.empty(na + 1, dtype=torch.float64, device=dev)
        DB = torch.empty(nb + 1, dtype=torch.float64, device=dev)
        flag = torch.ones(1, dtype=torch.int32, device=dev)
        st = torch.cuda.current_stream(dev).cuda_stream
        _lib.check(fn(ins[0].data_ptr(), ins[1].data_ptr(), na, ins[2].data_ptr(), ins[3].data_ptr(),
                      nb, d, 0.5, 0.25, 2, VA.data_ptr(), TA_.data_ptr(), DA.data_ptr(),
                      VB.data_ptr(), TB_.data_ptr(), DB.data_ptr(), flag.data_ptr(), ctypes.c_void_p(st)))
        torch.cuda.synchronize()
        assert flag.item() == 0
        for x, t, V, Tm, De, n in ((a, ta, VA, TA_, DA, na), (b, tb, VB, TB_, DB, nb)):
            ev, et, de = oracle.prepare_series(x.astype(np.float64), t.astype(np.float64), 0.5, 0.25, 2)
            V = V.cpu().numpy().astype(np.float64).reshape(n + 1, d)
            assert np.all(np.isinf(V[0])) and Tm[0].item() == 0.0 and math.isinf(De[0].item())
            assert np.array_equal(V[1:], ev[1:])
            assert np.array_equal(Tm.cpu().numpy().astype(np.float64), et)
            got = De.cpu().numpy()[1:]
            if f32:  # deletion costs of the fp32 mode: fp32-rounded inputs, fp64 arithmetic
                np.testing.assert_allclose(got, de[1:], rtol=1e-12)
            else:
                assert np.array_equal(got, de[1:])
    # the fused input check raises the flag for a NaN, an infinity, a huge value
    for bad in (np.nan, np.inf, 1e300 if not f32 else 1e30):
        a[na // 2, 0] = bad
        ins[0].copy_(torch.from_numpy(a.reshape(-1)))
        flag.zero_()
        _lib.check(fn(ins[0].data_ptr(), ins[1].data_ptr(), na, ins[2].data_ptr(), ins[3].data_ptr(),
                      nb, d, 0.5, 0.25, 2, VA.data_ptr(), TA_.data_ptr(), DA.data_ptr(),
                      VB.data_ptr(), TB_.data_ptr(), DB.data_ptr(), flag.data_ptr(), ctypes.c_void_p(st)))
        torch.cuda.synchronize()
        assert flag.item() == 1, bad
