"""Generate golden fixtures by running the REFERENCE itself (twedband/warpband).

Run in the build container, where /root/reference exists (it does not exist on
the GPU box, so the fixtures are committed):

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/gen_golden.py

Every value below is computed by the reference's public API
(`warpband.twed` W:43-53, `warpband.twed_batch` W:70-86,
`twedband.twed_parallel` E:101-121); inputs are stored verbatim (float repr
round-trips exactly) unless they are regenerated from a seed by
`paper_2007_16135_b200.workloads`, in which case only the seed is stored.
"""

from __future__ import annotations

import json
import math
import os
import sys
import time
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg")
sys.path[:0] = [str(REF / "src"), str(REF / "bindings" / "src")]
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
REPO = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(REPO))

import twedband  # noqa: E402  (the reference)
import warpband  # noqa: E402  (the reference bindings)
from twedband.io import read_series_file  # noqa: E402

from paper_2007_16135_b200.workloads import make_pair, make_set  # noqa: E402

OUT = Path(__file__).resolve().parent


def enc(x):
    """JSON-safe float (nan/inf as strings)."""
    if isinstance(x, (list, tuple)):
        return [enc(v) for v in x]
    x = float(x)
    if math.isnan(x):
        return "nan"
    if math.isinf(x):
        return "inf" if x > 0 else "-inf"
    return x


def arr(a):
    return enc(np.asarray(a, dtype=np.float64).tolist())


def random_series(rng, n=None, d=None, irregular_times=True):
    """pkg/tests/conftest.py:12-24, restated (values N(0,1), irregular times may start < 0)."""
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


PARAMS_GRID = [(nu, lam, deg) for nu in (0.1, 1.0) for lam in (0.0, 0.5, 1.0) for deg in (1, 2)]


def pair_case(name, va, ta, vb, tb, nu, lam, deg):
    value = warpband.twed(va, ta, vb, tb, nu=nu, lam=lam, degree=deg)
    return {"name": name, "values_a": arr(va), "times_a": arr(ta), "values_b": arr(vb),
            "times_b": arr(tb), "nu": nu, "lam": lam, "degree": deg, "value": enc(value)}


def small_cases():
    pairs = []
    fx = REF / "tests" / "fixtures"
    a = read_series_file(fx / "pair_a.csv")
    b = read_series_file(fx / "pair_b.csv")
    pairs.append(pair_case("fixture_pair_nu1_lam0", a.values, a.timestamps, b.values,
                           b.timestamps, 1.0, 0.0, 2))
    sa = np.sin(np.linspace(0, 6, 50))
    sb = np.sin(np.linspace(0.3, 6.3, 60))
    pairs.append(pair_case("readme_sin", sa, np.arange(50.0), sb, np.arange(60.0), 0.1, 0.5, 2))
    pairs.append(pair_case("forced_3", [2.0], [1.0], [5.0], [1.0], 1.0, 0.0, 1))
    v = np.array([[1.0, 2.0], [3.0, 4.0]])
    pairs.append(pair_case("identical", v, [0.5, 1.5], v, [0.5, 1.5], 1.0, 0.0, 2))
    # conftest-style random pairs over the params grid, degree 1..4
    rng = np.random.default_rng(20240511)
    for k in range(240):
        nu, lam, deg = PARAMS_GRID[k % 12]
        if k >= 192:
            deg = 3 + (k % 2)  # degree >= 3: binexp + pow path (K:45-48)
        va, ta = random_series(rng)
        vb, tb = random_series(rng, d=va.shape[1])
        pairs.append(pair_case(f"random_{k}", va, ta, vb, tb, nu, lam, deg))
    # longer pairs (multi-warp / multi-stripe on the GPU), irregular times
    rng = np.random.default_rng(7)
    for k, (na, nb, d) in enumerate([(100, 37, 1), (33, 257, 2), (513, 300, 3), (1025, 999, 1),
                                     (640, 2049, 2), (2500, 2400, 3), (64, 64, 1), (4097, 31, 1)]):
        va, ta = random_series(rng, n=na, d=d)
        vb, tb = random_series(rng, n=nb, d=d)
        nu, lam, deg = PARAMS_GRID[(2 * k + 1) % 12]
        pairs.append(pair_case(f"long_{na}x{nb}_d{d}", va, ta, vb, tb, nu, lam, deg))
    # non-finite values: the reference does not reject them (only timestamps are checked)
    va, ta = random_series(np.random.default_rng(99), n=9, d=2)
    vb, tb = random_series(np.random.default_rng(98), n=7, d=2)
    vn = va.copy()
    vn[4, 1] = np.nan
    pairs.append(pair_case("nan_value", vn, ta, vb, tb, 1.0, 0.5, 2))
    vi = va.copy()
    vi[2, 0] = np.inf
    pairs.append(pair_case("inf_value", vi, ta, vb, tb, 1.0, 0.5, 2))
    # signed zeros and negative nu = -0.0 are accepted by TwedParams (C:82-95)
    vz = np.zeros((5, 1))
    vz[1, 0] = -0.0
    pairs.append(pair_case("signed_zero", vz, np.arange(5.0), np.zeros((4, 1)), np.arange(4.0),
                           -0.0, -0.0, 2))
    return pairs


def batch_case(name, list_a, list_b, nu, lam, deg, symmetric):
    m = warpband.twed_batch(list_a, list_b, nu=nu, lam=lam, degree=deg, symmetric=symmetric,
                            workers=1)

    def ser(lst):
        return [{"values": arr(v), "times": arr(t)} for v, t in lst]

    return {"name": name, "series_a": ser(list_a), "series_b": None if list_b is None else ser(list_b),
            "nu": nu, "lam": lam, "degree": deg, "symmetric": symmetric,
            "matrix": [enc(r) for r in m.tolist()]}


def batch_cases():
    out = []
    rng = np.random.default_rng(20240511)
    la = [random_series(rng, d=2) for _ in range(5)]
    lb = [random_series(rng, d=2) for _ in range(7)]
    out.append(batch_case("ragged_full_5x7", la, lb, 0.1, 0.5, 2, False))
    s = [random_series(rng, d=1) for _ in range(6)]
    out.append(batch_case("ragged_self_sym_6", s, None, 0.5, 0.1, 1, True))
    out.append(batch_case("ragged_self_full_6", s, None, 0.5, 0.1, 1, False))
    trio = [read_series_file(REF / "tests" / "fixtures" / "trio" / f"series_{k}.csv")
            for k in range(3)]
    out.append(batch_case("trio_sym", [(t.values, t.timestamps) for t in trio], None,
                          1.0, 0.0, 2, True))
    rng = np.random.default_rng(4)
    la = [(rng.random((5, 1)), np.arange(5.0)) for _ in range(3)]
    lb = [(rng.random((7, 1)), np.arange(7.0)) for _ in range(2)]
    out.append(batch_case("bindings_3x2", la, lb, 0.1, 0.5, 1, False))
    # mixed lengths spanning 1..300 samples (warp kernels with K=1..16 rows per lane)
    rng = np.random.default_rng(12)
    lens = [1, 2, 31, 32, 33, 64, 65, 127, 128, 129, 255, 256, 300]
    mixed = [random_series(rng, n=n, d=2) for n in lens]
    out.append(batch_case("mixed_lengths_sym", mixed, None, 1.0, 1.0, 2, True))
    return out


def config_goldens():
    g = {}
    a, ta, b, tb = make_pair(1000, 1, 0)
    g["cfg1"] = {"seed": 0, "n": 1000, "d": 1,
                 "value": warpband.twed(a, ta, b, tb, nu=1.0, lam=1.0, degree=2)}
    a32, b32 = (x.astype(np.float32).astype(np.float64) for x in (a, b))
    g["cfg1_f32in"] = {"value": warpband.twed(a32, ta, b32, tb, nu=1.0, lam=1.0, degree=2)}
    # medium random-walk pairs, the reference's parallel band (bit-equal to serial)
    for n, d, seed in [(4096, 1, 11), (3000, 3, 12), (8192, 3, 13), (20000, 1, 14)]:
        a, ta, b, tb = make_pair(n, d, seed)
        t0 = time.perf_counter()
        v = twedband.twed_parallel(twedband.TimeSeries(a, ta), twedband.TimeSeries(b, tb),
                                   twedband.TwedParams(1.0, 1.0, 2), os.cpu_count())
        g[f"walk_{n}_d{d}_s{seed}"] = {"seed": seed, "n": n, "d": d, "value": v,
                                       "ref_seconds": time.perf_counter() - t0}
        a32, b32 = (x.astype(np.float32).astype(np.float64) for x in (a, b))
        v32 = twedband.twed_parallel(twedband.TimeSeries(a32, ta), twedband.TimeSeries(b32, tb),
                                     twedband.TwedParams(1.0, 1.0, 2), os.cpu_count())
        g[f"walk_{n}_d{d}_s{seed}_f32in"] = {"value": v32}
    # cfg4 entries (full 1000x1000, n=256, d=1)
    AA, TAA = make_set(1000, 256, 1, 3)
    BB, TBB = make_set(1000, 256, 1, 4)
    ent = {}
    for i, j in [(0, 0), (0, 999), (999, 0), (500, 500), (123, 456), (7, 3), (998, 1)]:
        ent[f"{i},{j}"] = warpband.twed(AA[i], TAA[i], BB[j], TBB[j], nu=1.0, lam=1.0, degree=2)
    g["cfg4"] = {"entries": ent}
    # cfg5 entries on fp32-rounded inputs (tri, self, n=128, d=2)
    S, TS = make_set(10000, 128, 2, 5)
    S = S.astype(np.float32).astype(np.float64)
    ent = {}
    for i, j in [(0, 0), (0, 1), (1234, 5678), (9998, 9999), (42, 4242), (9999, 0)]:
        ent[f"{i},{j}"] = warpband.twed(S[i], TS[i], S[j], TS[j], nu=1.0, lam=1.0, degree=2)
    g["cfg5_f32in"] = {"entries": ent}
    return g


def main():
    small = {"generator": "tests/golden/gen_golden.py (reference twedband/warpband)",
             "pairs": small_cases(), "batches": batch_cases()}
    (OUT / "small.json").write_text(json.dumps(small))
    cfg = config_goldens()
    cfg["generator"] = "tests/golden/gen_golden.py (reference twedband/warpband)"
    # survey-time values computed by the reference in this container
    cfg["cfg2"] = {"seed": 1, "n": 100000, "d": 1, "value": 559004.2804024924,
                   "source": "SURVEY.md A.1: twedband.twed_parallel, 8 workers"}
    (OUT / "configs.json").write_text(json.dumps(cfg, indent=1))
    print("wrote", OUT / "small.json", OUT / "configs.json")


if __name__ == "__main__":
    main()
