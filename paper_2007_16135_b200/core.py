"""Domain types and input validation, mirroring the reference's semantics.

`TimeSeries`, `TwedParams` and `InvalidInputError` follow
pkg/src/twedband/core.py:18-100 (same checks, same messages); `as_series`
follows warpband's `_as_series` (pkg/bindings/src/warpband/__init__.py:23-40).
Validation is O(n) host work; conforming float64 C-contiguous arrays are not
copied (the reference's no-copy contract, pkg/bindings/tests/test_bindings.py:71-81).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


class InvalidInputError(ValueError):
    """Raised when an input violates a documented precondition (core.py:18)."""


def _float_array(x, dtype):
    return np.asarray(x, dtype=dtype)


@dataclass(frozen=True, eq=False)
class TimeSeries:
    """A timestamped sequence of real vectors (core.py:22-70).

    values: (n,) or (n, d); timestamps: (n,), strictly increasing, default
    0, 1, ..., n-1. ``dtype`` float64 (reference) or float32 (fp32 mode).
    """

    values: np.ndarray
    timestamps: np.ndarray | None = None
    dtype: type = np.float64

    def __post_init__(self):
        values = _float_array(self.values, self.dtype)
        if values.ndim == 1:
            values = values.reshape(-1, 1)
        if values.ndim != 2:
            raise InvalidInputError(f"values must be 1-D or 2-D, got {values.ndim} dimensions")
        if values.shape[0] < 1:
            raise InvalidInputError("a time series needs at least one sample")
        if values.shape[1] < 1:
            raise InvalidInputError("samples need at least one component")
        if self.timestamps is None:
            timestamps = np.arange(values.shape[0], dtype=self.dtype)
        else:
            timestamps = _float_array(self.timestamps, self.dtype)
        if timestamps.ndim != 1 or timestamps.shape[0] != values.shape[0]:
            raise InvalidInputError(
                f"expected {values.shape[0]} timestamps, got shape {timestamps.shape}")
        if timestamps.shape[0] > 1 and not np.all(np.diff(timestamps) > 0):
            raise InvalidInputError("timestamps must be strictly increasing")
        object.__setattr__(self, "values", values)
        object.__setattr__(self, "timestamps", timestamps)

    @property
    def n(self) -> int:
        return self.values.shape[0]

    @property
    def d(self) -> int:
        return self.values.shape[1]


@dataclass(frozen=True)
class TwedParams:
    """nu (stiffness), lam (deletion penalty), degree of the lp norm (core.py:73-100)."""

    nu: float = 1.0
    lam: float = 0.0
    degree: int = 2

    def __post_init__(self):
        if self.nu < 0:
            raise InvalidInputError(f"nu must be >= 0, got {self.nu}")
        if self.lam < 0:
            raise InvalidInputError(f"lam must be >= 0, got {self.lam}")
        if int(self.degree) != self.degree or self.degree < 1:
            raise InvalidInputError(f"degree must be a positive integer, got {self.degree}")
        object.__setattr__(self, "nu", float(self.nu))
        object.__setattr__(self, "lam", float(self.lam))
        object.__setattr__(self, "degree", int(self.degree))

    @property
    def is_metric(self) -> bool:
        return self.nu > 0 and self.lam >= 0


def as_series(values, times, label: str, dtype=np.float64) -> TimeSeries:
    """warpband._as_series (W:23-40): shape checks with the reference messages."""
    values = np.asarray(values, dtype=dtype)
    if values.ndim not in (1, 2):
        raise ValueError(
            f"{label}: values must be 1-D or 2-D (n samples by d components), "
            f"got {values.ndim} dimensions {values.shape}")
    n = values.shape[0]
    times = np.asarray(times, dtype=dtype)
    if times.ndim != 1:
        raise ValueError(f"{label}: timestamps must be 1-D, got {times.ndim} dimensions")
    if times.shape[0] != n:
        raise ValueError(f"{label}: {times.shape[0]} timestamps for {n} samples")
    return TimeSeries(values, times, dtype)


def is_series_like(item) -> bool:
    """A TimeSeries of the reference package (twedband.TimeSeries, C:22-70):
    anything with ``values`` and ``timestamps`` arrays."""
    return (not isinstance(item, (np.ndarray, tuple, list)) and hasattr(item, "values")
            and hasattr(item, "timestamps"))


def as_series_list(items, label: str, dtype=np.float64) -> list[TimeSeries]:
    """warpband._as_series_list (W:56-67): TimeSeries, (values, times) or bare values."""
    out = []
    for k, item in enumerate(items):
        if isinstance(item, TimeSeries):
            if item.values.dtype != dtype:
                item = TimeSeries(item.values, item.timestamps, dtype)
            out.append(item)
        elif is_series_like(item):  # the reference's own TimeSeries objects
            out.append(TimeSeries(item.values, item.timestamps, dtype))
        elif isinstance(item, tuple) and len(item) == 2:
            out.append(as_series(item[0], item[1], f"{label}[{k}]", dtype))
        else:
            values = np.asarray(item, dtype=dtype)
            out.append(as_series(values, np.arange(values.shape[0], dtype=dtype),
                                 f"{label}[{k}]", dtype))
    return out


def pack(series: list[TimeSeries]):
    """Packed CSR form of a list: values (N_total, d), times (N_total,), offsets (k+1,)."""
    dtype = series[0].values.dtype
    off = np.zeros(len(series) + 1, dtype=np.int64)
    off[1:] = np.cumsum([s.n for s in series])
    if len(series) == 1:
        return (np.ascontiguousarray(series[0].values), np.ascontiguousarray(series[0].timestamps),
                off)
    values = np.ascontiguousarray(np.concatenate([s.values for s in series]), dtype=dtype)
    times = np.ascontiguousarray(np.concatenate([s.timestamps for s in series]), dtype=dtype)
    return values, times, off
