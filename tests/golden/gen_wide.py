"""Golden fixtures for series with d >= 5 components, computed by the REFERENCE.

The reference's lp_dist loops over any number of components
(pkg/src/twedband/_kernels.py:24-48) and the paper benchmarks R^28 series
(MNIST 60k x 60k, n = 28). Run in the build container,
where /root/reference exists:

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/gen_wide.py

Writes tests/golden/wide.json (pair values; inputs regenerated from the stored
seeds by tests/golden/series.py or paper_2007_16135_b200.workloads) and
tests/golden/wide_batches.npz (batch matrices; inputs from the seeds in
wide.json's "batches").
Every value comes from the reference's public API (warpband.twed W:43-53,
warpband.twed_batch W:70-86).
"""

from __future__ import annotations

import json
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
sys.path.insert(0, str(Path(__file__).resolve().parent))

import warpband  # noqa: E402  (the reference bindings)

from gen_golden import enc, PARAMS_GRID  # noqa: E402
from series import ragged_set, seeded_pair  # noqa: E402
from paper_2007_16135_b200.workloads import make_pair, make_set  # noqa: E402

OUT = Path(__file__).resolve().parent


# batch workloads regenerated from seeds by the tests (kept in sync with them)
BATCHES = {
    # MNIST-shaped: 200 series of 28 samples in R^28, symmetric (tri)
    "mnist_like_200_tri": dict(kind="set", count=200, n=28, d=28, seed=6, nu=1.0, lam=1.0,
                               degree=2, symmetric=True),
    # ragged d = 5, full A x B
    "ragged_d5_full": dict(kind="ragged", seed_a=21, lengths_a=[1, 7, 33, 64, 65, 128, 129, 200],
                           seed_b=22, lengths_b=[3, 31, 32, 100, 256, 17], d=5, nu=0.5, lam=0.25,
                           degree=2, symmetric=False),
    # d = 8, degree 1, ragged self batch, symmetric
    "ragged_d8_sym_p1": dict(kind="ragged", seed_a=23, lengths_a=[5, 40, 90, 130, 255, 12, 70],
                             seed_b=None, lengths_b=None, d=8, nu=1.0, lam=0.5, degree=1,
                             symmetric=True),
    # rows longer than 256 samples (the wavefront per pair), d = 6
    "long_rows_d6": dict(kind="ragged", seed_a=24, lengths_a=[300, 520, 64], seed_b=25,
                         lengths_b=[280, 40, 700], d=6, nu=1.0, lam=1.0, degree=2,
                         symmetric=False),
}


def batch_inputs(spec):
    if spec["kind"] == "set":
        S, T = make_set(spec["count"], spec["n"], spec["d"], spec["seed"])
        return [(S[k], T[k]) for k in range(spec["count"])], None
    la = ragged_set(spec["seed_a"], spec["lengths_a"], spec["d"])
    lb = None if spec["seed_b"] is None else ragged_set(spec["seed_b"], spec["lengths_b"], spec["d"])
    return la, lb


def pair_case(name, spec, nu, lam, deg):
    va, ta, vb, tb = seeded_pair(spec)
    value = warpband.twed(va, ta, vb, tb, nu=nu, lam=lam, degree=deg)
    return {"name": name, "inputs": spec, "nu": nu, "lam": lam, "degree": deg,
            "value": enc(value)}


def pairs():
    out = []
    seed = 1000
    for d in (5, 8, 28):
        lens = np.random.default_rng(d).integers(1, 40, size=(24, 2))
        for k in range(24):
            nu, lam, deg = PARAMS_GRID[k % 12]
            if k >= 20:
                deg = 3 + (k % 2)
            spec = {"seed": seed, "na": int(lens[k, 0]), "nb": int(lens[k, 1]), "d": d}
            seed += 1
            out.append(pair_case(f"random_d{d}_{k}", spec, nu, lam, deg))
    # longer pairs: several warps / stripes / CTAs of the wavefront
    for k, (na, nb, d) in enumerate([(300, 257, 5), (1025, 700, 8), (640, 1500, 28),
                                     (2600, 2500, 5), (64, 3000, 12)]):
        nu, lam, deg = PARAMS_GRID[(2 * k + 1) % 12]
        spec = {"seed": 2000 + k, "na": na, "nb": nb, "d": d}
        out.append(pair_case(f"long_{na}x{nb}_d{d}", spec, nu, lam, deg))
    # non-finite values (not rejected by the reference; the NaN-exact min)
    out.append(pair_case("nan_value_d6", {"seed": 97, "na": 30, "nb": 25, "d": 6,
                                          "poke": [[11, 4, "nan"]]}, 1.0, 0.5, 2))
    out.append(pair_case("inf_value_d6", {"seed": 97, "na": 30, "nb": 25, "d": 6,
                                          "poke": [[3, 5, "inf"]]}, 1.0, 0.5, 2))
    # random walks with unit times (the benchmark generator), d = 8
    a, ta, b, tb = make_pair(4000, 8, 31)
    out.append({"name": "walk_4000_d8", "walk": {"n": 4000, "d": 8, "seed": 31}, "nu": 1.0,
                "lam": 1.0, "degree": 2,
                "value": enc(warpband.twed(a, ta, b, tb, nu=1.0, lam=1.0, degree=2))})
    return out


def main():
    t0 = time.perf_counter()
    data = {"generator": "tests/golden/gen_wide.py (reference twedband/warpband)",
            "pairs": pairs(), "batches": BATCHES}
    (OUT / "wide.json").write_text(json.dumps(data))
    mats = {}
    for name, spec in BATCHES.items():
        la, lb = batch_inputs(spec)
        m = warpband.twed_batch(la, lb, nu=spec["nu"], lam=spec["lam"], degree=spec["degree"],
                                symmetric=spec["symmetric"], workers=os.cpu_count())
        mats[name] = np.asarray(m, dtype=np.float64)
    np.savez_compressed(OUT / "wide_batches.npz", **mats)
    print(f"wrote wide.json, wide_batches.npz in {time.perf_counter() - t0:.1f} s")


if __name__ == "__main__":
    main()
