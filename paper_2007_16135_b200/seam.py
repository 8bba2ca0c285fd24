"""Kernel-seam adapter: the reference package's band solvers on the B200 kernels.

The reference engine looks its band solvers up as module attributes at call
time (pkg/src/twedband/engine.py:20,77,91), with the S2 signature of
pkg/src/twedband/_kernels.py:128,146

    twed_band_serial(z, z1, z2, va, ta, del_a, vb, tb, del_b, nu, p) -> float
    twed_band_parallel(z, z1, z2, va, ta, del_a, vb, tb, del_b, nu, p) -> float

on the prepared (zero-prefixed) arrays of core.prepare_series
(pkg/src/twedband/core.py:218-234). ``band_solve`` below has that signature
and runs the sweep through ``twb_band_solve_f64`` (include/twb.h). ``install``
swaps it into a ``twedband`` module so every reference caller -- warpband.twed,
twedband.twed_parallel, twedband.twed_batch, the CLI -- runs on the GPU, and
the reference's own test-suite can be pointed at the GPU kernel unchanged
(scripts/ref_seam_plugin.py, scripts/run_reference_suite.sh,
tests/test_gpu_reference_suite.py).

``z``, ``z1``, ``z2`` are the reference's scratch diagonals; the GPU sweep
keeps its band on the device and does not touch them (the value returned is
the reference's ``z[nb]``).
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib

_pd = ctypes.POINTER(ctypes.c_double)


def _c64(x):
    a = np.ascontiguousarray(x, dtype=np.float64)
    return a


def band_solve(z, z1, z2, va, ta, del_a, vb, tb, del_b, nu, p, device=0) -> float:
    """S2 seam (_kernels.py:127-174) on libtwb200: returns the band's z[nb]."""
    lib = _lib.load()
    va, vb = _c64(va), _c64(vb)
    if va.ndim == 1:
        va = va.reshape(-1, 1)
    if vb.ndim == 1:
        vb = vb.reshape(-1, 1)
    ta, del_a, tb, del_b = (_c64(x) for x in (ta, del_a, tb, del_b))
    out = ctypes.c_double(0.0)
    _lib.check(lib.twb_band_solve_f64(
        va.ctypes.data_as(_pd), ta.ctypes.data_as(_pd), del_a.ctypes.data_as(_pd),
        va.shape[0] - 1, vb.ctypes.data_as(_pd), tb.ctypes.data_as(_pd),
        del_b.ctypes.data_as(_pd), vb.shape[0] - 1, va.shape[1], float(nu), int(p),
        int(device), ctypes.byref(out)))
    return float(out.value)


def lcs_solve(z, z1, z2, s, t, device=0) -> int:
    """S2 seam for LCS (_kernels.py:193-219, lcs_band_solve) on libtwb200: the
    int64 symbol codes of core._encode_symbols in, the LCS length out."""
    from .api import lcs_codes
    return lcs_codes(s, t, device=device)


class Installed:
    """Handle returned by ``install``; ``restore()`` puts the CPU kernels back."""

    def __init__(self, kernels, saved):
        self.kernels = kernels
        self.saved = saved
        self.calls = 0

    def restore(self):
        for name, fn in self.saved.items():
            setattr(self.kernels, name, fn)


class _Saved:
    """Attributes replaced on several modules, restorable."""

    def __init__(self):
        self.items = []

    def swap(self, module, name, fn):
        self.items.append((module, name, getattr(module, name)))
        setattr(module, name, fn)

    def restore(self):
        for module, name, fn in reversed(self.items):
            setattr(module, name, fn)
        self.items.clear()


def install(twedband_module=None, device=0, batch=False) -> Installed:
    """Point ``twedband._kernels.twed_band_serial/_parallel`` (and
    ``lcs_band_solve``) at the GPU sweeps.

    batch=True also routes ``twedband.twed_batch`` / ``twedband.engine.twed_batch``
    (E:183-226) to ONE all-pairs kernel launch on the GPU, instead of one
    band-solve call (two host synchronisations) per pair: same entries, same
    symmetric layout, the reference's DistanceMatrix. It is off by default
    because the reference's own tests count the per-pair solver calls of its
    batch (T/test_engine.py:127-128)."""
    if twedband_module is None:
        import twedband as twedband_module  # the reference package
    kernels = twedband_module._kernels
    _lib.require_device()
    names = ("twed_band_serial", "twed_band_parallel")
    if hasattr(kernels, "lcs_band_solve"):  # present in the reference; optional here
        names += ("lcs_band_solve",)
    saved = {name: getattr(kernels, name) for name in names}
    handle = Installed(kernels, saved)
    if batch:
        engine = twedband_module.engine
        extra = _Saved()

        def gpu_twed_batch(spec):
            from .api import batch_matrix
            from .core import TimeSeries, TwedParams
            handle.calls += 1
            mk = lambda lst: [TimeSeries(s.values, s.timestamps) for s in lst]  # noqa: E731
            list_a = mk(spec.list_a)
            list_b = None if spec.is_self_batch else mk(spec.list_b)
            p = spec.params
            out = batch_matrix(list_a, list_b, TwedParams(p.nu, p.lam, p.degree),
                               symmetric=spec.symmetric, device=device)
            return engine.DistanceMatrix(entries=out, symmetric=spec.symmetric)

        extra.swap(engine, "twed_batch", gpu_twed_batch)
        if getattr(twedband_module, "twed_batch", None) is not None:
            extra.swap(twedband_module, "twed_batch", gpu_twed_batch)
        base_restore = handle.restore

        def restore():
            extra.restore()
            base_restore()
        handle.restore = restore

    def gpu_band(z, z1, z2, va, ta, del_a, vb, tb, del_b, nu, p):
        handle.calls += 1
        return band_solve(z, z1, z2, va, ta, del_a, vb, tb, del_b, nu, p, device=device)

    def gpu_lcs(z, z1, z2, s, t):
        handle.calls += 1
        return lcs_solve(z, z1, z2, s, t, device=device)

    kernels.twed_band_serial = gpu_band
    kernels.twed_band_parallel = gpu_band
    if "lcs_band_solve" in saved:
        kernels.lcs_band_solve = gpu_lcs
    return handle
