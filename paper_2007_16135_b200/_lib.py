"""ctypes binding of the C ABI in include/twb.h (libtwb200.so, sm_100a).

There is no CPU fallback: if the shared library is missing or no CUDA device
is visible, every compute entry point raises. ``ctypes`` releases the GIL for
the duration of each call, like the reference's ``nogil`` numba kernels
(pkg/src/twedband/_kernels.py:24-127).
"""

from __future__ import annotations

import ctypes
import os
import threading
from pathlib import Path

PKG_DIR = Path(__file__).resolve().parent
LIB_PATH = PKG_DIR / "lib" / "libtwb200.so"

TWB_OK, TWB_EINVAL, TWB_ECUDA, TWB_ENOMEM, TWB_EUNSUP = 0, -1, -2, -3, -4

_d = ctypes.c_double
_f = ctypes.c_float
_i32 = ctypes.c_int32
_i64 = ctypes.c_int64
_pd = ctypes.POINTER(ctypes.c_double)
_pf = ctypes.POINTER(ctypes.c_float)
_pi64 = ctypes.POINTER(ctypes.c_int64)
_pi32 = ctypes.POINTER(ctypes.c_int32)
_vp = ctypes.c_void_p

_SIGS = {
    "twb_version": (ctypes.c_int, []),
    "twb_last_error": (ctypes.c_size_t, [ctypes.c_char_p, ctypes.c_size_t]),
    "twb_device_count": (ctypes.c_int, []),
    "twb_take_launch_count": (_i64, []),
    "twb_set_kernel_timing": (None, [ctypes.c_int]),
    "twb_last_kernel_ms": (ctypes.c_float, []),
    "twb_last_wave_shape": (None, [_pi64, _pi64, _pi64]),
    "twb_probe_add_rate": (ctypes.c_double, [ctypes.c_int, ctypes.c_int]),
    "twb_selftest_sqrt": (_i64, [_i64, ctypes.c_uint64, _i32, ctypes.POINTER(_i64)]),
    "twb_twed_f64": (ctypes.c_int, [_pd, _i64, _pd, _pd, _i64, _pd, _i32, _d, _d, _i32, _i32, _pd]),
    "twb_twed_f32": (ctypes.c_int, [_pf, _i64, _pf, _pf, _i64, _pf, _i32, _d, _d, _i32, _i32, _pd]),
    "twb_twed_multi_f64": (ctypes.c_int, [_pd, _i64, _pd, _pd, _i64, _pd, _i32, _d, _d, _i32, _pi32,
                                          _i32, _pd]),
    "twb_twed_multi_f32": (ctypes.c_int, [_pf, _i64, _pf, _pf, _i64, _pf, _i32, _d, _d, _i32, _pi32,
                                          _i32, _pd]),
    "twb_lcs_i32": (ctypes.c_int, [_pi32, _i64, _pi32, _i64, _i32, _i32, _pi64]),
    "twb_twed_dev_f64": (ctypes.c_int, [_vp, _i64, _vp, _vp, _i64, _vp, _i32, _d, _d, _i32, _vp, _vp]),
    "twb_twed_dev_f32": (ctypes.c_int, [_vp, _i64, _vp, _vp, _i64, _vp, _i32, _d, _d, _i32, _vp, _vp]),
    "twb_twed_batch_f64": (ctypes.c_int, [_pd, _pi64, _i64, _pd, _pd, _pi64, _i64, _pd, _i32, _d, _d,
                                          _i32, _i32, _i64, _i64, _i32, _pd]),
    "twb_twed_batch_f32": (ctypes.c_int, [_pf, _pi64, _i64, _pf, _pf, _pi64, _i64, _pf, _i32, _d, _d,
                                          _i32, _i32, _i64, _i64, _i32, _pf]),
    "twb_twed_batch_multi_f64": (ctypes.c_int, [_pd, _pi64, _i64, _pd, _pd, _pi64, _i64, _pd, _i32,
                                                _d, _d, _i32, _i32, _pi32, _i32, _pd]),
    "twb_twed_batch_multi_f32": (ctypes.c_int, [_pf, _pi64, _i64, _pf, _pf, _pi64, _i64, _pf, _i32,
                                                _d, _d, _i32, _i32, _pi32, _i32, _pf]),
    "twb_twed_batch_dev_f64": (ctypes.c_int, [_vp, _pi64, _i64, _vp, _vp, _pi64, _i64, _vp, _i32, _d,
                                              _d, _i32, _i32, _i64, _i64, _vp, _vp]),
    "twb_twed_batch_dev_f32": (ctypes.c_int, [_vp, _pi64, _i64, _vp, _vp, _pi64, _i64, _vp, _i32, _d,
                                              _d, _i32, _i32, _i64, _i64, _vp, _vp]),
    "twb_mirror_upper_dev_f64": (ctypes.c_int, [_vp, _i64, _vp]),
    "twb_mirror_upper_dev_f32": (ctypes.c_int, [_vp, _i64, _vp]),
    "twb_band_solve_f64": (ctypes.c_int, [_pd, _pd, _pd, _i64, _pd, _pd, _pd, _i64, _i32, _d, _i32,
                                          _i32, _pd]),
    "twb_prepare_series_f64": (ctypes.c_int, [_pd, _pd, _i64, _i32, _d, _d, _i32, _i32, _pd, _pd,
                                              _pd]),
    "twb_prepare_pair_dev_f64": (ctypes.c_int, [_vp, _vp, _i64, _vp, _vp, _i64, _i32, _d, _d, _i32,
                                                _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "twb_prepare_pair_dev_f32": (ctypes.c_int, [_vp, _vp, _i64, _vp, _vp, _i64, _i32, _d, _d, _i32,
                                                _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "twb_trim_pool": (ctypes.c_int, [_i32]),
}

_lock = threading.Lock()
_lib = None


class TwbError(RuntimeError):
    """A CUDA-side failure reported by libtwb200 (reference: none, CPU only)."""


def load():
    """Load libtwb200.so (raises if it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            path = Path(os.environ.get("TWB_LIBRARY", LIB_PATH))
            if not path.exists():
                raise ImportError(
                    f"libtwb200.so not found at {path}; build it with "
                    "`python -c 'import __graft_entry__ as g; g.build()'` "
                    "(make -C paper_2007_16135_b200/csrc)")
            lib = ctypes.CDLL(str(path))
            variant = "TWB_LIBRARY" in os.environ  # A/B builds may predate newer entry points
            for name, (res, args) in _SIGS.items():
                if variant and not hasattr(lib, name):
                    continue
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    return _lib


def exported_symbols():
    return sorted(_SIGS)


def last_error() -> str:
    lib = load()
    buf = ctypes.create_string_buffer(2048)
    lib.twb_last_error(buf, len(buf))
    return buf.value.decode(errors="replace")


def check(rc: int) -> None:
    if rc == TWB_OK:
        return
    msg = last_error()
    if rc in (TWB_EINVAL,):
        raise ValueError(msg)
    if rc == TWB_EUNSUP:
        raise NotImplementedError(msg)
    if rc == TWB_ENOMEM:
        raise MemoryError(msg)
    raise TwbError(msg)


def device_count() -> int:
    try:
        return int(load().twb_device_count())
    except ImportError:
        return 0


def take_launch_count() -> int:
    return int(load().twb_take_launch_count())


def require_device() -> None:
    """Raise loudly when there is no CUDA device: there is no CPU path."""
    if device_count() < 1:
        raise TwbError("no CUDA device visible: libtwb200 has no CPU fallback "
                       "(run on a B200, e.g. via gpurun)")
