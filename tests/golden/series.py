"""Seeded input generators shared by the golden generators and the tests
(no reference import: the tests regenerate fixture inputs from stored seeds).

``random_series`` restates the reference suite's fixture
(pkg/tests/conftest.py:12-24): N(0, 1) values and irregular timestamps that
may start below 0.
"""

from __future__ import annotations

import numpy as np


def random_series(rng, n=None, d=None, irregular_times=True):
    if n is None:
        n = int(rng.integers(1, 24))
    if d is None:
        d = int(rng.integers(1, 4))
    values = rng.standard_normal((n, d))
    if irregular_times:
        start = rng.uniform(-5.0, 5.0)
        times = start + np.cumsum(rng.uniform(0.05, 2.0, size=n))
    else:
        times = np.arange(n, dtype=np.float64)
    return values, times


def seeded_pair(spec):
    """Inputs of a wide.json pair case: {"seed", "na", "nb", "d"} (+ optional
    "poke": [[row, col, value], ...] applied to A)."""
    rng = np.random.default_rng(spec["seed"])
    va, ta = random_series(rng, n=spec["na"], d=spec["d"])
    vb, tb = random_series(rng, n=spec["nb"], d=spec["d"])
    for r, c, v in spec.get("poke", []):
        va[r, c] = float(v)
    return va, ta, vb, tb


def ragged_set(seed, lengths, d):
    rng = np.random.default_rng(seed)
    return [random_series(rng, n=n, d=d) for n in lengths]
