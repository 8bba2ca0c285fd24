"""Drop-in for the reference bindings ``warpband`` (pkg/bindings/src/warpband/__init__.py).

Same signatures, defaults, validation and messages as the reference module;
values come from the B200 kernels. ``workers`` is validated like the
reference's ``resolve_workers`` (pkg/src/twedband/engine.py:42-62) and then
ignored: the GPU, not a CPU thread pool, runs the pairs.
"""

from __future__ import annotations

import os

from .api import batch_matrix, twed_series
from .core import InvalidInputError, TwedParams, as_series, as_series_list

__all__ = ["twed", "twed_batch", "resolve_workers"]

WORKERS_ENV = "WARPBAND_WORKERS"


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
        raise InvalidInputError(f"workers must be an integer or 'auto', got {workers!r}")
    if workers < 1:
        raise InvalidInputError(f"workers must be >= 1, got {workers}")
    return workers


def twed(values_a, times_a, values_b, times_b, nu=1.0, lam=0.0, degree=2) -> float:
    """warpband.twed (W:43-53)."""
    a = as_series(values_a, times_a, "series A")
    b = as_series(values_b, times_b, "series B")
    if a.d != b.d:
        raise ValueError(f"series dimensions differ: A has d={a.d}, B has d={b.d}")
    return twed_series(a, b, TwedParams(nu=nu, lam=lam, degree=degree))


def twed_batch(series_a, series_b=None, *, nu=1.0, lam=0.0, degree=2, symmetric=False,
               workers="auto"):
    """warpband.twed_batch (W:70-86): lists of TimeSeries / (values, times) / values."""
    params = TwedParams(nu=nu, lam=lam, degree=degree)
    resolve_workers(workers)
    list_a = as_series_list(series_a, "series_a")
    if series_b is None:
        list_b = None
    else:
        list_b = as_series_list(series_b, "series_b")
        # BatchSpec.is_self_batch (E:171-175): the same objects in the same order
        same = len(list_a) == len(list_b) and all(x is y for x, y in zip(list_a, list_b))
        if same:
            list_b = None
        elif symmetric:
            raise InvalidInputError("symmetric=True requires both lists to be the same collection")
    if not list_a or (list_b is not None and not list_b):
        raise InvalidInputError("batch lists must be nonempty")
    return batch_matrix(list_a, list_b, params, symmetric=symmetric)
