"""TEST INFRASTRUCTURE ONLY — ctypes front-end of the CPU parity oracle.

Wraps ``oracle/_build/liboracle.so`` (built from ``oracle/twed_oracle.c`` by
``oracle/Makefile``), the operation-for-operation C restatement of the
reference ``twedband`` kernels (pkg/src/twedband/_kernels.py:24-174,
core.py:218-234, engine.py:101-226). Only ``tests/``, ``__graft_entry__.smoke``
and ``bench.py`` (cpu_baseline leg and ``--impl reference``) may import this
module, and only as the checker / the timed CPU comparator. The product package
``paper_2007_16135_b200`` never imports it.

Parity pinning: ``tests/test_oracle_golden.py`` checks this oracle bit-for-bit
against fixtures produced by the reference itself (``tests/golden/gen_golden.py``).
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB_PATH = HERE / "_build" / "liboracle.so"

_c_double_p = ctypes.POINTER(ctypes.c_double)
_c_int64_p = ctypes.POINTER(ctypes.c_int64)
_lib = None


def build(force: bool = False) -> Path:
    """Compile the oracle with the committed Makefile (gcc, -ffp-contract=off)."""
    src = HERE / "twed_oracle.c"
    if force or not LIB_PATH.exists() or LIB_PATH.stat().st_mtime < src.stat().st_mtime:
        subprocess.run(["make", "-s", "-C", str(HERE)], check=True)
    return LIB_PATH


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(str(LIB_PATH))
        lib.orc_lp_dist.restype = ctypes.c_double
        lib.orc_lp_dist.argtypes = [_c_double_p, _c_double_p, ctypes.c_int, ctypes.c_int64]
        lib.orc_prepare_series.restype = None
        lib.orc_prepare_series.argtypes = [
            _c_double_p, _c_double_p, ctypes.c_int64, ctypes.c_int, ctypes.c_double,
            ctypes.c_double, ctypes.c_int64, _c_double_p, _c_double_p, _c_double_p,
        ]
        band = [_c_double_p, _c_double_p, _c_double_p, ctypes.c_int64,
                _c_double_p, _c_double_p, _c_double_p, ctypes.c_int64,
                ctypes.c_int, ctypes.c_double, ctypes.c_int64]
        lib.orc_band_serial.restype = ctypes.c_double
        lib.orc_band_serial.argtypes = band
        lib.orc_band_parallel.restype = ctypes.c_double
        lib.orc_band_parallel.argtypes = band + [ctypes.c_int]
        lib.orc_band_tiled.restype = ctypes.c_double
        lib.orc_band_tiled.argtypes = band + [ctypes.c_int, ctypes.c_int]
        lib.orc_fill_matrix.restype = None
        lib.orc_fill_matrix.argtypes = [_c_double_p] + band
        lib.orc_twed.restype = ctypes.c_double
        lib.orc_twed.argtypes = [
            _c_double_p, _c_double_p, ctypes.c_int64, _c_double_p, _c_double_p, ctypes.c_int64,
            ctypes.c_int, ctypes.c_double, ctypes.c_double, ctypes.c_int64, ctypes.c_int,
        ]
        lib.orc_twed_batch.restype = ctypes.c_int
        lib.orc_lcs_band.restype = ctypes.c_int64
        lib.orc_lcs_band.argtypes = [ctypes.POINTER(ctypes.c_int64), ctypes.c_int64,
                                     ctypes.POINTER(ctypes.c_int64), ctypes.c_int64]
        lib.orc_twed_batch.argtypes = [
            _c_double_p, _c_double_p, _c_int64_p, ctypes.c_int64,
            _c_double_p, _c_double_p, _c_int64_p, ctypes.c_int64,
            ctypes.c_int, ctypes.c_double, ctypes.c_double, ctypes.c_int64,
            ctypes.c_int, ctypes.c_int, _c_double_p,
        ]
        lib.orc_max_threads.restype = ctypes.c_int
        _lib = lib
    return _lib


def _f64(x, ndim=None):
    a = np.ascontiguousarray(np.asarray(x, dtype=np.float64))
    if ndim == 2 and a.ndim == 1:
        a = a.reshape(-1, 1)
    return a


def _p(a):
    return a.ctypes.data_as(_c_double_p)


def max_threads() -> int:
    return int(_load().orc_max_threads())


def lp_dist(x, y, p: int) -> float:
    x, y = _f64(x).reshape(-1), _f64(y).reshape(-1)
    return float(_load().orc_lp_dist(_p(x), _p(y), x.shape[0], int(p)))


def prepare_series(values, times, nu: float, lam: float, degree: int):
    """(ext_values (n+1,d), ext_times (n+1,), deletion (n+1,)) — core.py:218-234."""
    v = _f64(values, 2)
    t = _f64(times)
    n, d = v.shape
    ev = np.empty((n + 1, d))
    et = np.empty(n + 1)
    de = np.empty(n + 1)
    _load().orc_prepare_series(_p(v), _p(t), n, d, float(nu), float(lam), int(degree),
                               _p(ev), _p(et), _p(de))
    return ev, et, de


def band_serial(pa, pb, nu: float, degree: int) -> float:
    """twed_band_serial on prepared arrays — _kernels.py:127-142."""
    (va, ta, da), (vb, tb, db) = pa, pb
    return float(_load().orc_band_serial(
        _p(va), _p(ta), _p(da), va.shape[0] - 1, _p(vb), _p(tb), _p(db), vb.shape[0] - 1,
        va.shape[1], float(nu), int(degree)))


def band_tiled(pa, pb, nu: float, degree: int, threads: int = 0, tile: int = 256) -> float:
    """Bit-identical tiled schedule of the same band (fast golden generation)."""
    (va, ta, da), (vb, tb, db) = pa, pb
    return float(_load().orc_band_tiled(
        _p(va), _p(ta), _p(da), va.shape[0] - 1, _p(vb), _p(tb), _p(db), vb.shape[0] - 1,
        va.shape[1], float(nu), int(degree), int(threads), int(tile)))


def twed_tiled(values_a, times_a, values_b, times_b, nu=1.0, lam=0.0, degree=2, threads=0,
               tile=256) -> float:
    pa = prepare_series(values_a, times_a, nu, lam, degree)
    pb = prepare_series(values_b, times_b, nu, lam, degree)
    return band_tiled(pa, pb, nu, degree, threads, tile)


def fill_matrix(pa, pb, nu: float, degree: int) -> np.ndarray:
    """Full (na+1, nb+1) cost matrix — _kernels.py:83-97 / reference.py:17-41."""
    (va, ta, da), (vb, tb, db) = pa, pb
    dp = np.empty((va.shape[0], vb.shape[0]))
    _load().orc_fill_matrix(
        _p(dp), _p(va), _p(ta), _p(da), va.shape[0] - 1, _p(vb), _p(tb), _p(db),
        vb.shape[0] - 1, va.shape[1], float(nu), int(degree))
    return dp


def twed(values_a, times_a, values_b, times_b, nu=1.0, lam=0.0, degree=2, threads=1) -> float:
    """Distance of one pair — engine.py:101-121 (threads>1 -> parallel band)."""
    a, b = _f64(values_a, 2), _f64(values_b, 2)
    ta, tb = _f64(times_a), _f64(times_b)
    if a.shape[1] != b.shape[1]:
        raise ValueError("series dimensions differ")
    return float(_load().orc_twed(_p(a), _p(ta), a.shape[0], _p(b), _p(tb), b.shape[0],
                                  a.shape[1], float(nu), float(lam), int(degree), int(threads)))


def _pack(series):
    vals = [_f64(v, 2) for v, _ in series]
    times = [_f64(t) for _, t in series]
    off = np.zeros(len(vals) + 1, dtype=np.int64)
    off[1:] = np.cumsum([v.shape[0] for v in vals])
    return np.ascontiguousarray(np.concatenate(vals)), np.ascontiguousarray(np.concatenate(times)), off


def twed_batch(series_a, series_b=None, nu=1.0, lam=0.0, degree=2, symmetric=False,
               threads=0) -> np.ndarray:
    """All-pairs matrix — engine.py:183-226. series_* are lists of (values, times)."""
    va, ta, oa = _pack(series_a)
    d = va.shape[1]
    out = np.empty((len(series_a), len(series_a if series_b is None else series_b)))
    lib = _load()
    if series_b is None:
        rc = lib.orc_twed_batch(_p(va), _p(ta), oa.ctypes.data_as(_c_int64_p), len(series_a),
                                None, None, None, 0, d, float(nu), float(lam), int(degree),
                                int(bool(symmetric)), int(threads), _p(out))
    else:
        vb, tb, ob = _pack(series_b)
        rc = lib.orc_twed_batch(_p(va), _p(ta), oa.ctypes.data_as(_c_int64_p), len(series_a),
                                _p(vb), _p(tb), ob.ctypes.data_as(_c_int64_p), len(series_b),
                                d, float(nu), float(lam), int(degree), int(bool(symmetric)),
                                int(threads), _p(out))
    if rc != 0:
        raise MemoryError("oracle batch allocation failed")
    return out


def host_description() -> dict:
    model = ""
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"cpu_count": os.cpu_count(), "model": model, "omp_threads": max_threads()}


def encode_symbols(s, t):
    """core._encode_symbols (C:141-160): strings -> code points, other
    sequences -> one shared first-seen code table."""
    if isinstance(s, str) and isinstance(t, str):
        return (np.array([ord(c) for c in s], dtype=np.int64),
                np.array([ord(c) for c in t], dtype=np.int64))
    codes = {}

    def enc(seq):
        return np.array([codes.setdefault(x, len(codes)) for x in list(seq)], dtype=np.int64)

    return enc(s), enc(t)


def lcs(s, t) -> int:
    """LCS length, band.lcs_band (band.py:185-197) -> _kernels.lcs_band_solve (K:193-219)."""
    a, b = encode_symbols(s, t) if not isinstance(s, np.ndarray) else (
        np.ascontiguousarray(s, dtype=np.int64), np.ascontiguousarray(t, dtype=np.int64))
    pi = ctypes.POINTER(ctypes.c_int64)
    r = _load().orc_lcs_band(a.ctypes.data_as(pi), a.size, b.ctypes.data_as(pi), b.size)
    if r < 0:
        raise MemoryError("oracle: out of memory")
    return int(r)
