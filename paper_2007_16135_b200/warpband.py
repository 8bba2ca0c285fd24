"""Drop-in for the reference bindings ``warpband`` (pkg/bindings/src/warpband/__init__.py).

Same names, signatures, defaults, validation and messages as the reference
module (``twed``, ``twed_batch``, ``lcs_length``, ``__version__``, and the
``_as_series`` helper its tests use); values come from the B200 kernels.
``workers`` is validated like the reference's ``resolve_workers``
(pkg/src/twedband/engine.py:42-62) and then ignored: the GPU, not a CPU thread
pool, runs the pairs.

Errors: validation failures raise ``InvalidInputError`` (a ``ValueError``).
When the reference package ``twedband`` is importable, the exception raised
is also an instance of ``twedband.InvalidInputError`` (core.py:18), so
reference callers' ``except twedband.InvalidInputError`` keep working; the
reference is imported only on that error path.
"""

from __future__ import annotations

import functools
import os
import sys

from . import core
from .api import batch_matrix, lcs, twed_series
from .core import TwedParams, as_series, as_series_list

__all__ = ["twed", "twed_batch", "lcs_length", "resolve_workers", "__version__"]

# Version of the reference bindings' API this module implements
# (pkg/src/twedband/__init__.py:41; the bindings re-export it, W:18).
__version__ = "0.1.0"

WORKERS_ENV = "WARPBAND_WORKERS"

_compat_error = None


def _error_class():
    """core.InvalidInputError, or a subclass that is also the reference's
    twedband.InvalidInputError when the reference package is importable."""
    global _compat_error
    if _compat_error is None:
        base = None
        ref = sys.modules.get("twedband")
        try:
            if ref is None:
                import twedband as ref  # noqa: PLC0415  (error path only)
            base = getattr(ref, "InvalidInputError", None)
        except Exception:  # reference not installed: our own class is the contract
            base = None
        if isinstance(base, type) and issubclass(base, Exception) and \
                not issubclass(core.InvalidInputError, base):
            _compat_error = type("InvalidInputError", (core.InvalidInputError, base),
                                 {"__module__": __name__})
        else:
            _compat_error = core.InvalidInputError
    return _compat_error


def __getattr__(name):
    if name == "InvalidInputError":
        return _error_class()
    raise AttributeError(name)


def _reference_errors(fn):
    @functools.wraps(fn)
    def wrapper(*args, **kwargs):
        try:
            return fn(*args, **kwargs)
        except core.InvalidInputError as exc:
            cls = _error_class()
            if isinstance(exc, cls):
                raise
            raise cls(*exc.args) from None
    return wrapper


def resolve_workers(workers=None) -> int:
    """engine.resolve_workers (E:42-62): None/'auto' -> env or cpu_count."""
    if workers in (None, "auto"):
        env = os.environ.get(WORKERS_ENV)
        if env is not None:
            workers = env
        else:
            return os.cpu_count() or 1
    try:
        if int(workers) != float(workers):
            raise ValueError
        workers = int(workers)
    except (TypeError, ValueError):
        raise core.InvalidInputError(f"workers must be an integer or 'auto', got {workers!r}")
    if workers < 1:
        raise core.InvalidInputError(f"workers must be >= 1, got {workers}")
    return workers


@_reference_errors
def _as_series(values, times, label: str):
    """warpband._as_series (W:23-40): shape checks, no copy of conforming arrays."""
    return as_series(values, times, label)


@_reference_errors
def twed(values_a, times_a, values_b, times_b, nu=1.0, lam=0.0, degree=2) -> float:
    """warpband.twed (W:43-53)."""
    a = as_series(values_a, times_a, "series A")
    b = as_series(values_b, times_b, "series B")
    if a.d != b.d:
        raise ValueError(f"series dimensions differ: A has d={a.d}, B has d={b.d}")
    return twed_series(a, b, TwedParams(nu=nu, lam=lam, degree=degree))


@_reference_errors
def twed_batch(series_a, series_b=None, *, nu=1.0, lam=0.0, degree=2, symmetric=False,
               workers="auto"):
    """warpband.twed_batch (W:70-86): lists of TimeSeries / (values, times) / values."""
    params = TwedParams(nu=nu, lam=lam, degree=degree)
    resolve_workers(workers)
    list_a = as_series_list(series_a, "series_a")
    if series_b is None:
        list_b = None  # BatchSpec.self_batch (E:177-180)
    else:
        # BatchSpec.is_self_batch (E:171-175): the same TimeSeries objects in
        # the same order (tuples / arrays become new series, never "the same")
        same = len(series_a) == len(series_b) and all(
            x is y and _is_series(x) for x, y in zip(series_a, series_b))
        list_b = None if same else as_series_list(series_b, "series_b")
    # BatchSpec.__post_init__ (E:155-169), in its order
    if not list_a or (list_b is not None and not list_b):
        raise core.InvalidInputError("batch lists must be nonempty")
    dim = list_a[0].d
    for s in list(list_a) + list(list_b or []):
        if s.d != dim:
            raise core.InvalidInputError(f"batch series dimensions differ: {s.d} vs {dim}")
    if symmetric and list_b is not None:
        raise core.InvalidInputError("symmetric=True requires both lists to be the same collection")
    return batch_matrix(list_a, list_b, params, symmetric=symmetric)


def _is_series(x) -> bool:
    return isinstance(x, core.TimeSeries) or core.is_series_like(x)


def lcs_length(s, t) -> int:
    """warpband.lcs_length (W:89-91): longest-common-subsequence length of two
    strings (twedband.lcs_band), on the bit-parallel GPU sweep."""
    return lcs(s, t)
