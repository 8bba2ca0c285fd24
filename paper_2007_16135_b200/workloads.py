"""Synthetic workloads of BASELINE.json's configs.

Random-walk series with unit-spaced timestamps (the reference default,
pkg/src/twedband/core.py:50-51 in TimeSeries.__post_init__). Parameters for
every config: nu=1.0, lam=1.0, degree=2.
"""

from __future__ import annotations

import numpy as np

PARAMS = {"nu": 1.0, "lam": 1.0, "degree": 2}


def make_pair(n: int, d: int, seed: int):
    """A then B from one generator: cumsum of standard normals, T = 0..n-1."""
    rng = np.random.default_rng(seed)
    a = np.cumsum(rng.standard_normal((n, d)), axis=0)
    b = np.cumsum(rng.standard_normal((n, d)), axis=0)
    t = np.arange(n, dtype=np.float64)
    return a, t, b, t.copy()


def make_set(count: int, n: int, d: int, seed: int):
    """(count, n, d) random walks and (count, n) unit-spaced timestamps."""
    rng = np.random.default_rng(seed)
    values = np.cumsum(rng.standard_normal((count, n, d)), axis=1)
    times = np.broadcast_to(np.arange(n, dtype=np.float64), (count, n)).copy()
    return values, times


# BASELINE.json "configs", in order.
CONFIGS = {
    "cfg1": dict(kind="pair", n=1_000, d=1, seed=0, dtype="f64"),
    "cfg2": dict(kind="pair", n=100_000, d=1, seed=1, dtype="f64"),
    "cfg3": dict(kind="pair", n=1_000_000, d=3, seed=2, dtype="f64"),
    "cfg3_f32": dict(kind="pair", n=1_000_000, d=3, seed=2, dtype="f32"),
    "cfg4": dict(kind="batch", count_a=1_000, count_b=1_000, n=256, d=1, seed_a=3, seed_b=4,
                 tri=False, dtype="f64"),
    "cfg5": dict(kind="batch", count_a=10_000, n=128, d=2, seed_a=5, tri=True, dtype="f32"),
}
