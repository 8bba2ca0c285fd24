"""Public API: the reference path's functions on the B200 library.

North-star spellings (cuTWED style) and the reference package's spellings are
both accepted:

    twed(A, TA, B, TB, nu=1.0, lamb=0.0, degree=2)          # == warpband.twed(..., lam=)
    twed_batch(AA, TAA, BB, TBB, nu, lamb, degree, tri)      # == warpband.twed_batch(
                                                             #    series_a, series_b, symmetric=)

Reference seams replaced:
    twed          -> warpband.twed                 pkg/bindings/src/warpband/__init__.py:43-53
                     twedband.engine.twed_parallel pkg/src/twedband/engine.py:101-121
    twed_batch    -> warpband.twed_batch           pkg/bindings/src/warpband/__init__.py:70-86
                     twedband.engine.twed_batch    pkg/src/twedband/engine.py:183-226
    band_solve    -> twedband._kernels.twed_band_serial / _parallel (prepared arrays)
                                                   pkg/src/twedband/_kernels.py:127-174
    prepare_series-> twedband.core.prepare_series  pkg/src/twedband/core.py:218-234

Precision: ``dtype=np.float64`` (default, bit-identical to the reference) or
``dtype=np.float32`` (fp32 inputs, fp32 local costs; the DP accumulates in
fp64 for long series; within 1e-5 relative of the fp64 reference on the same
fp32-rounded inputs).
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from .core import (
    InvalidInputError,
    TimeSeries,
    TwedParams,
    as_series,
    as_series_list,
    pack,
)

_pd = ctypes.POINTER(ctypes.c_double)
_pf = ctypes.POINTER(ctypes.c_float)
_pi64 = ctypes.POINTER(ctypes.c_int64)


def _ptr(a):
    if a is None:
        return None
    return a.ctypes.data_as(_pd if a.dtype == np.float64 else _pf)


def _lam(lamb, lam):
    if lam is not None and lamb is not None and float(lam) != float(lamb):
        raise TypeError("pass the deletion penalty once: lamb= (cuTWED) or lam= (warpband)")
    value = lam if lam is not None else lamb
    return 0.0 if value is None else value


def _dtype(dtype):
    if dtype is None:
        return np.float64
    dt = np.dtype(dtype)
    if dt not in (np.dtype(np.float64), np.dtype(np.float32)):
        raise ValueError(f"dtype must be float64 or float32, got {dt}")
    return dt.type


def twed(A, TA, B, TB, nu=1.0, lamb=None, degree=2, *, lam=None, dtype=None, device=0) -> float:
    """Time warp edit distance between two timestamped series.

    ``A``/``B`` have shape (n,) or (n, d) with matching d; ``TA``/``TB`` shape
    (n,), strictly increasing. Same validation and messages as warpband.twed.
    """
    dt = _dtype(dtype)
    a = as_series(A, TA, "series A", dt)
    b = as_series(B, TB, "series B", dt)
    if a.d != b.d:
        raise ValueError(f"series dimensions differ: A has d={a.d}, B has d={b.d}")
    params = TwedParams(nu=nu, lam=_lam(lamb, lam), degree=degree)
    return twed_series(a, b, params, device=device)


def twed_series(a: TimeSeries, b: TimeSeries, params: TwedParams, device=0) -> float:
    """engine.twed_parallel equivalent on validated series (E:101-121).

    ``device`` is one CUDA device, or a sequence of devices: the pair's
    wavefront then runs as one ring of CTAs over one kernel per listed device
    (twb_twed_multi_*; a device may repeat). Same result, bit for bit."""
    if a.d != b.d:
        raise InvalidInputError(f"series dimensions differ: {a.d} vs {b.d}")
    lib = _lib.load()
    _lib.require_device()
    va, ta = np.ascontiguousarray(a.values), np.ascontiguousarray(a.timestamps)
    vb, tb = np.ascontiguousarray(b.values), np.ascontiguousarray(b.timestamps)
    out = ctypes.c_double(0.0)
    f64 = va.dtype == np.float64
    if isinstance(device, (list, tuple, np.ndarray)):
        devs = np.ascontiguousarray(device, dtype=np.int32)
        if devs.ndim != 1 or devs.size < 1:
            raise ValueError("device list must be a non-empty 1-D sequence")
        fn = lib.twb_twed_multi_f64 if f64 else lib.twb_twed_multi_f32
        _lib.check(fn(_ptr(va), a.n, _ptr(ta), _ptr(vb), b.n, _ptr(tb), a.d, params.nu,
                      params.lam, params.degree, devs.ctypes.data_as(_lib._pi32), int(devs.size),
                      ctypes.byref(out)))
        return float(out.value)
    fn = lib.twb_twed_f64 if f64 else lib.twb_twed_f32
    _lib.check(fn(_ptr(va), a.n, _ptr(ta), _ptr(vb), b.n, _ptr(tb), a.d, params.nu, params.lam,
                  params.degree, int(device), ctypes.byref(out)))
    return float(out.value)


class _Packed:
    """A validated list of series in packed CSR form (what pack() returns)
    built straight from stacked (N, n[, d]) arrays: one vectorised check of
    every series (TimeSeries.__post_init__'s rules, C:37-62) and no per-series
    objects or copies -- a 10k-series list costs microseconds, not a Python loop."""

    def __init__(self, X, T, label, dt):
        X = np.asarray(X, dtype=dt)
        if X.ndim == 2:
            X = X[:, :, None]
        N, n, d = X.shape
        if N < 1:
            raise InvalidInputError("batch lists must be nonempty")
        if n < 1:
            raise InvalidInputError("a time series needs at least one sample")
        if d < 1:
            raise InvalidInputError("samples need at least one component")
        if T is None:
            T = np.broadcast_to(np.arange(n, dtype=dt), (N, n))
        T = np.asarray(T, dtype=dt)
        if T.shape != (N, n):
            raise ValueError(f"{label}: timestamps shape {T.shape} does not match values {(N, n)}")
        if n > 1 and not np.all(T[:, 1:] > T[:, :-1]):
            raise InvalidInputError("timestamps must be strictly increasing")
        self.values = np.ascontiguousarray(X.reshape(N * n, d))
        self.times = np.ascontiguousarray(T.reshape(N * n))
        self.off = np.arange(N + 1, dtype=np.int64) * n
        self.count, self.d = N, d

    def __len__(self):
        return self.count


def _to_list(X, T, label, dt):
    if isinstance(X, np.ndarray) or (hasattr(X, "shape") and not isinstance(X, (list, tuple))):
        arr = np.asarray(X)
        if arr.ndim in (2, 3) and (T is None or np.asarray(T).ndim == 2):
            return _Packed(arr, T, label, dt)
    items = list(X)
    if T is not None:
        times = list(T)
        if len(times) != len(items):
            raise ValueError(f"{label}: {len(times)} timestamp arrays for {len(items)} series")
        items = [(v, t) for v, t in zip(items, times)]
    return as_series_list(items, label, dt)


def batch_matrix(list_a, list_b, params: TwedParams, symmetric=False, device=0,
                 row_begin=0, row_end=None) -> np.ndarray:
    """engine.twed_batch (E:183-226) on validated lists. list_b None -> self batch.

    Returns the (row_end - row_begin) x len(list_b) block of rows
    [row_begin, row_end) of the distance matrix (all rows by default). With
    symmetric=True and all rows, the full mirrored matrix (E:223-225).
    """
    if not len(list_a) or (list_b is not None and not len(list_b)):
        raise InvalidInputError("batch lists must be nonempty")

    def packed(lst):  # (values, times, offsets, d)
        if isinstance(lst, _Packed):
            return lst.values, lst.times, lst.off, lst.d
        dims = {s.d for s in lst}
        if len(dims) > 1:
            raise InvalidInputError(f"batch series dimensions differ: {sorted(dims)}")
        return (*pack(lst), lst[0].d)

    va, ta, oa, dim = packed(list_a)
    lib = _lib.load()
    _lib.require_device()
    nA = len(list_a)
    if row_end is None:
        row_end = nA
    if list_b is None:
        vb = tb = ob = None
        nB = nA
    else:
        vb, tb, ob, dim_b = packed(list_b)
        if dim_b != dim:
            raise InvalidInputError(f"batch series dimensions differ: {dim_b} vs {dim}")
        nB = len(list_b)
    f32 = va.dtype == np.float32
    out = np.empty((row_end - row_begin, nB), dtype=np.float32 if f32 else np.float64)
    fn = lib.twb_twed_batch_f32 if f32 else lib.twb_twed_batch_f64

    def solve(r0, r1, dev, dst):
        _lib.check(fn(_ptr(va), oa.ctypes.data_as(_pi64), nA, _ptr(ta), _ptr(vb),
                      None if ob is None else ob.ctypes.data_as(_pi64), nB, _ptr(tb), dim,
                      params.nu, params.lam, params.degree, int(bool(symmetric)), int(r0),
                      int(r1), int(dev), _ptr(dst)))

    if not isinstance(device, (list, tuple, np.ndarray)):
        solve(row_begin, row_end, device, out)
        return out
    # Several devices: one C call (twb_twed_batch_multi_*) shards contiguous
    # row blocks balanced by work over the devices, one host thread each, no
    # collective; every device writes its rows -- and for the triangle the
    # transposed mirror of its rows' upper part, made on the device -- straight
    # into `out` (engine.py:200-203, 223-225).
    devs = np.ascontiguousarray([int(d) for d in device], dtype=np.int32)
    if devs.size == 0:
        raise ValueError("device list must be non-empty")
    if row_begin != 0 or row_end != nA:
        raise ValueError("a device list computes the whole matrix (no row range)")
    fm = lib.twb_twed_batch_multi_f32 if f32 else lib.twb_twed_batch_multi_f64
    _lib.check(fm(_ptr(va), oa.ctypes.data_as(_pi64), nA, _ptr(ta), _ptr(vb),
                  None if ob is None else ob.ctypes.data_as(_pi64), nB, _ptr(tb), dim,
                  params.nu, params.lam, params.degree, int(bool(symmetric)),
                  devs.ctypes.data_as(_lib._pi32), int(devs.size), _ptr(out)))
    return out


def twed_batch(AA, TAA=None, BB=None, TBB=None, nu=1.0, lamb=None, degree=2, tri=None, *,
               lam=None, symmetric=None, dtype=None, device=0) -> np.ndarray:
    """All-pairs distance matrix R[i, j] = twed(AA[i], BB[j]).

    AA / BB: stacked (N, n) or (N, n, d) arrays with (N, n) timestamps TAA /
    TBB (None -> 0, 1, ..., n-1), or lists of series (values arrays, (values,
    times) tuples or TimeSeries) with TAA / TBB None or lists of timestamps.
    BB None -> self batch (the only case where tri / symmetric is allowed).
    tri (= the reference's symmetric=True): solve j >= i and mirror, same
    output as the full matrix.
    """
    if tri is not None and symmetric is not None and bool(tri) != bool(symmetric):
        raise TypeError("pass the triangle flag once: tri= (cuTWED) or symmetric= (warpband)")
    sym = bool(tri if tri is not None else (symmetric or False))
    dt = _dtype(dtype)
    params = TwedParams(nu=nu, lam=_lam(lamb, lam), degree=degree)
    list_a = _to_list(AA, TAA, "series_a", dt)
    list_b = None if BB is None else _to_list(BB, TBB, "series_b", dt)
    if sym and list_b is not None:
        raise InvalidInputError("symmetric=True requires both lists to be the same collection")
    if not len(list_a):
        raise InvalidInputError("batch lists must be nonempty")
    return batch_matrix(list_a, list_b, params, symmetric=sym, device=device)


def band_solve(pa, pb, nu: float, degree: int, device=0) -> float:
    """_kernels.twed_band_serial / twed_band_parallel seam (K:127-174).

    pa / pb = (ext_values (n+1, d), ext_times (n+1,), deletion (n+1,)), the
    reference's PreparedSeries arrays (C:177-234).
    """
    lib = _lib.load()
    _lib.require_device()
    (va, ta, da), (vb, tb, db) = pa, pb
    va = np.ascontiguousarray(va, dtype=np.float64)
    vb = np.ascontiguousarray(vb, dtype=np.float64)
    if va.ndim == 1:
        va = va.reshape(-1, 1)
    if vb.ndim == 1:
        vb = vb.reshape(-1, 1)
    ta, da, tb, db = (np.ascontiguousarray(x, dtype=np.float64) for x in (ta, da, tb, db))
    out = ctypes.c_double(0.0)
    _lib.check(lib.twb_band_solve_f64(_ptr(va), _ptr(ta), _ptr(da), va.shape[0] - 1, _ptr(vb),
                                      _ptr(tb), _ptr(db), vb.shape[0] - 1, va.shape[1], float(nu),
                                      int(degree), int(device), ctypes.byref(out)))
    return float(out.value)


def prepare_series(series: TimeSeries, params: TwedParams, device=0):
    """core.prepare_series (C:218-234) on the GPU: (ext_values, ext_times, deletion)."""
    lib = _lib.load()
    _lib.require_device()
    v = np.ascontiguousarray(series.values, dtype=np.float64)
    t = np.ascontiguousarray(series.timestamps, dtype=np.float64)
    ev = np.empty((series.n + 1, series.d))
    et = np.empty(series.n + 1)
    de = np.empty(series.n + 1)
    _lib.check(lib.twb_prepare_series_f64(_ptr(v), _ptr(t), series.n, series.d, params.nu,
                                          params.lam, params.degree, int(device), _ptr(ev),
                                          _ptr(et), _ptr(de)))
    return ev, et, de


# ---------------------------------------------------------------------------
# Device-resident variants (torch CUDA tensors in, torch CUDA tensor out),
# the paper's twed_dev: no host copies, caller's stream.
# ---------------------------------------------------------------------------
def _check_cuda(name, t, dtype, device, numel=None):
    """Device-resident arguments: a contiguous CUDA tensor of the given dtype
    on the given device (and size). A mismatch would otherwise read or write
    out of bounds on the device."""
    import torch

    if not isinstance(t, torch.Tensor):
        raise TypeError(f"{name} must be a torch.Tensor, got {type(t).__name__}")
    if not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor")
    if t.device != device:
        raise ValueError(f"{name} is on {t.device}, expected {device} (all tensors on one device)")
    if t.dtype != dtype:
        raise ValueError(f"{name} has dtype {t.dtype}, expected {dtype}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    if numel is not None and t.numel() != numel:
        raise ValueError(f"{name} has {t.numel()} elements, expected {numel}")


def twed_dev(A, TA, B, TB, nu=1.0, lamb=None, degree=2, *, lam=None, out=None, stream=None):
    """A, TA, B, TB: contiguous CUDA tensors (float64 or float32) on one device. Returns
    a 1-element float64 CUDA tensor (or fills ``out``). Validation of timestamps is the
    caller's responsibility (no host round trip); shapes, dtypes and devices are checked."""
    import torch

    params = TwedParams(nu=nu, lam=_lam(lamb, lam), degree=degree)
    lib = _lib.load()
    if not isinstance(A, torch.Tensor) or not isinstance(B, torch.Tensor):
        raise TypeError("twed_dev takes torch CUDA tensors")
    if A.dim() not in (1, 2) or B.dim() not in (1, 2):
        raise ValueError("values must be 1-D or 2-D (n samples by d components)")
    A2 = A if A.dim() == 2 else A.reshape(-1, 1)
    B2 = B if B.dim() == 2 else B.reshape(-1, 1)
    if A2.shape[1] != B2.shape[1]:
        raise ValueError(f"series dimensions differ: A has d={A2.shape[1]}, B has d={B2.shape[1]}")
    if A2.dtype not in (torch.float64, torch.float32):
        raise ValueError(f"values must be float64 or float32, got {A2.dtype}")
    dev = A2.device
    _check_cuda("A", A2, A2.dtype, dev)
    _check_cuda("B", B2, A2.dtype, dev)
    _check_cuda("TA", TA, A2.dtype, dev, A2.shape[0])
    _check_cuda("TB", TB, A2.dtype, dev, B2.shape[0])
    if A2.shape[0] < 1 or B2.shape[0] < 1:
        raise InvalidInputError("a time series needs at least one sample")
    if out is None:
        out = torch.empty(1, dtype=torch.float64, device=dev)
    _check_cuda("out", out, torch.float64, dev)
    if out.numel() < 1:
        raise ValueError("out needs one element")
    st = stream if stream is not None else torch.cuda.current_stream(dev)
    fn = lib.twb_twed_dev_f64 if A2.dtype == torch.float64 else lib.twb_twed_dev_f32
    with torch.cuda.device(dev):
        _lib.check(fn(A2.data_ptr(), A2.shape[0], TA.data_ptr(), B2.data_ptr(), B2.shape[0],
                      TB.data_ptr(), A2.shape[1], params.nu, params.lam, params.degree,
                      st.cuda_stream, out.data_ptr()))
    return out


def _check_offsets(name, off, rows):
    off = np.ascontiguousarray(off, dtype=np.int64)
    if off.ndim != 1 or off.shape[0] < 2:
        raise InvalidInputError("batch lists must be nonempty")
    if off[0] != 0:
        raise ValueError(f"{name}[0] must be 0, got {off[0]}")
    if np.any(np.diff(off) < 1):
        raise InvalidInputError("a time series needs at least one sample")
    if off[-1] != rows:
        raise ValueError(f"{name}[-1] = {off[-1]} does not match the {rows} packed samples")
    return off


def twed_batch_dev(AA, a_off, TAA, BB=None, b_off=None, TBB=None, nu=1.0, lamb=None, degree=2,
                   tri=False, *, lam=None, row_begin=0, row_end=None, out=None, stream=None):
    """Packed device inputs: AA (N_total, d) CUDA tensor, a_off host int64 CSR offsets
    (N+1,) starting at 0, TAA (N_total,). Returns the (row_end-row_begin, nB) block on the
    device (AA's dtype). Every tensor is checked (device, dtype, contiguity, size)."""
    import torch

    params = TwedParams(nu=nu, lam=_lam(lamb, lam), degree=degree)
    lib = _lib.load()
    if not isinstance(AA, torch.Tensor):
        raise TypeError("twed_batch_dev takes torch CUDA tensors")
    if AA.dim() not in (1, 2):
        raise ValueError("packed values must be 1-D or 2-D (samples by components)")
    AA2 = AA if AA.dim() == 2 else AA.reshape(-1, 1)
    if AA2.dtype not in (torch.float64, torch.float32):
        raise ValueError(f"values must be float64 or float32, got {AA2.dtype}")
    dev, dt = AA2.device, AA2.dtype
    dim = AA2.shape[1]
    _check_cuda("AA", AA2, dt, dev)
    a_off = _check_offsets("a_off", a_off, AA2.shape[0])
    _check_cuda("TAA", TAA, dt, dev, AA2.shape[0])
    nA = a_off.shape[0] - 1
    if (BB is None) != (TBB is None) or (BB is None) != (b_off is None):
        raise ValueError("pass BB, b_off and TBB together (or none of them for a self batch)")
    BB2 = None
    if BB is not None:
        if not isinstance(BB, torch.Tensor) or BB.dim() not in (1, 2):
            raise ValueError("BB must be a 1-D or 2-D CUDA tensor")
        BB2 = BB if BB.dim() == 2 else BB.reshape(-1, 1)
        if BB2.shape[1] != dim:
            raise InvalidInputError(f"batch series dimensions differ: {BB2.shape[1]} vs {dim}")
        _check_cuda("BB", BB2, dt, dev)
        b_off = _check_offsets("b_off", b_off, BB2.shape[0])
        _check_cuda("TBB", TBB, dt, dev, BB2.shape[0])
        nB = b_off.shape[0] - 1
        if tri:
            raise InvalidInputError("symmetric=True requires both lists to be the same collection")
    else:
        nB = nA
    if row_end is None:
        row_end = nA
    if not (0 <= row_begin < row_end <= nA):
        raise ValueError(f"row range [{row_begin}, {row_end}) outside [0, {nA})")
    if out is None:
        out = torch.empty((row_end - row_begin, nB), dtype=dt, device=dev)
    _check_cuda("out", out, dt, dev, (row_end - row_begin) * nB)
    st = stream if stream is not None else torch.cuda.current_stream(dev)
    fn = lib.twb_twed_batch_dev_f32 if dt == torch.float32 else lib.twb_twed_batch_dev_f64
    with torch.cuda.device(dev):
        _lib.check(fn(AA2.data_ptr(), a_off.ctypes.data_as(_pi64), nA, TAA.data_ptr(),
                      None if BB2 is None else BB2.data_ptr(),
                      None if BB2 is None else b_off.ctypes.data_as(_pi64), nB,
                      None if BB2 is None else TBB.data_ptr(), dim, params.nu, params.lam,
                      params.degree, int(bool(tri)), int(row_begin), int(row_end),
                      st.cuda_stream, out.data_ptr()))
    return out


def mirror_upper_dev(M, stream=None):
    """Mirror the strict upper triangle of a square CUDA matrix into its lower half."""
    import torch

    lib = _lib.load()
    st = stream if stream is not None else torch.cuda.current_stream(M.device)
    fn = lib.twb_mirror_upper_dev_f32 if M.dtype == torch.float32 else lib.twb_mirror_upper_dev_f64
    with torch.cuda.device(M.device):
        _lib.check(fn(M.data_ptr(), M.shape[0], st.cuda_stream))
    return M


# ---------------------------------------------------------------------------
# LCS length (band.lcs_band, pkg/src/twedband/band.py:185-197).
# ---------------------------------------------------------------------------
def _encode_symbols(s, t):
    """core._encode_symbols (C:141-160): strings use code points, other
    sequences of hashable symbols share one first-seen code table."""
    if isinstance(s, str) and isinstance(t, str):
        return (np.array([ord(c) for c in s], dtype=np.int64),
                np.array([ord(c) for c in t], dtype=np.int64))
    codes: dict = {}

    def encode(seq):
        out = np.empty(len(seq), dtype=np.int64)
        for i, sym in enumerate(seq):
            out[i] = codes.setdefault(sym, len(codes))
        return out

    return encode(list(s)), encode(list(t))


def lcs(s, t, device=0) -> int:
    """Longest-common-subsequence length of two strings or sequences of
    hashable symbols; empty inputs give 0 (reference: band.lcs_band). Runs the
    bit-parallel sweep of libtwb200 (twb_lcs_i32); integer-exact."""
    a, b = _encode_symbols(s, t)
    if a.size == 0 or b.size == 0:
        return 0
    _lib.require_device()
    return lcs_codes(a, b, device=device)


def dense_codes(a, b):
    """int64 symbol codes -> int32 codes in [0, A) for the A symbols present in
    both sequences, -1 for the rest (they can never match)."""
    a = np.asarray(a, dtype=np.int64)
    b = np.asarray(b, dtype=np.int64)
    common = np.intersect1d(a, b)
    if common.size == 0:
        return (np.full(a.size, -1, np.int32), np.full(b.size, -1, np.int32), 0)
    ia = np.minimum(np.searchsorted(common, a), common.size - 1)
    ib = np.minimum(np.searchsorted(common, b), common.size - 1)
    ca = np.where(common[ia] == a, ia, -1).astype(np.int32)
    cb = np.where(common[ib] == b, ib, -1).astype(np.int32)
    return np.ascontiguousarray(ca), np.ascontiguousarray(cb), int(common.size)


def lcs_codes(a, b, device=0) -> int:
    """LCS length of two int64 code sequences through twb_lcs_i32."""
    ca, cb, A = dense_codes(a, b)
    if ca.size == 0 or cb.size == 0:
        return 0
    lib = _lib.load()
    out = ctypes.c_int64(0)
    pi = ctypes.POINTER(ctypes.c_int32)
    _lib.check(lib.twb_lcs_i32(ca.ctypes.data_as(pi), ca.size, cb.ctypes.data_as(pi), cb.size,
                               A, int(device), ctypes.byref(out)))
    return int(out.value)
