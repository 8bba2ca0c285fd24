"""Pin the CPU oracle (oracle/twed_oracle.c) to the reference's own outputs.

The fixtures were produced by the reference itself (tests/golden/gen_golden.py
imports twedband/warpband); the oracle must reproduce them bit for bit for
degree 1 and 2 (sqrt is IEEE-exact) and within 1e-12 relative for degree>=3
(libm pow decides the last bits, pkg/src/twedband/_kernels.py:45-48).
"""

import json
import math

import numpy as np
import pytest

from conftest import (GOLDEN, as_values, dec, exact_expected, same_float, wide_batch_inputs,
                      wide_pair_inputs)
from paper_2007_16135_b200.workloads import make_pair, make_set


def test_pairs_bit_exact(small_golden, oracle):
    n_exact = 0
    for case in small_golden["pairs"]:
        got = oracle.twed(as_values(case["values_a"]), as_values(case["times_a"]),
                          as_values(case["values_b"]), as_values(case["times_b"]),
                          case["nu"], case["lam"], case["degree"])
        want = float(dec(case["value"]))
        if case["degree"] <= 2 or np.asarray(dec(case["values_a"])).ndim == 1 or \
                np.asarray(dec(case["values_a"])).shape[1] == 1:
            assert same_float(got, want), (case["name"], got, want)
            n_exact += 1
        else:
            assert got == pytest.approx(want, rel=1e-12), case["name"]
    assert n_exact > 200


def test_parallel_band_matches_serial(small_golden, oracle):
    for case in small_golden["pairs"]:
        if not case["name"].startswith("long_"):
            continue
        args = (as_values(case["values_a"]), as_values(case["times_a"]),
                as_values(case["values_b"]), as_values(case["times_b"]),
                case["nu"], case["lam"], case["degree"])
        assert same_float(oracle.twed(*args, threads=4), float(case["value"])), case["name"]


def test_tiled_schedule_matches_reference(small_golden, config_golden, oracle):
    """orc_band_tiled (the schedule that produced the n = 1M cfg3 golden,
    tests/golden/gen_cfg3.py) reproduces the reference's own values bit for bit."""
    n = 0
    for case in small_golden["pairs"]:
        if case["degree"] > 2:
            continue
        args = (as_values(case["values_a"]), as_values(case["times_a"]),
                as_values(case["values_b"]), as_values(case["times_b"]),
                case["nu"], case["lam"], case["degree"])
        for tile in (3, 64):
            got = oracle.twed_tiled(*args, threads=2, tile=tile)
            assert same_float(got, float(dec(case["value"]))), (case["name"], tile)
        n += 1
    assert n > 100
    a, ta, b, tb = make_pair(3000, 3, 12)  # reference value computed by twedband itself
    assert oracle.twed_tiled(a, ta, b, tb, 1.0, 1.0, 2, threads=4, tile=512) == \
        config_golden["walk_3000_d3_s12"]["value"]


def test_full_matrix_corner_matches_band(small_golden, oracle):
    for case in small_golden["pairs"][:60]:
        pa = oracle.prepare_series(as_values(case["values_a"]), as_values(case["times_a"]),
                                   case["nu"], case["lam"], case["degree"])
        pb = oracle.prepare_series(as_values(case["values_b"]), as_values(case["times_b"]),
                                   case["nu"], case["lam"], case["degree"])
        dp = oracle.fill_matrix(pa, pb, case["nu"], case["degree"])
        assert same_float(dp[-1, -1], oracle.band_serial(pa, pb, case["nu"], case["degree"]))


def _series(lst):
    return [(as_values(s["values"]), as_values(s["times"])) for s in lst]


def test_batches_bit_exact(small_golden, oracle):
    for case in small_golden["batches"]:
        la = _series(case["series_a"])
        lb = None if case["series_b"] is None else _series(case["series_b"])
        got = oracle.twed_batch(la, lb, case["nu"], case["lam"], case["degree"],
                                case["symmetric"], threads=4)
        want = np.asarray(dec(case["matrix"]))
        assert got.shape == want.shape
        assert np.array_equal(got, want), case["name"]


def test_config_goldens(config_golden, oracle):
    a, ta, b, tb = make_pair(1000, 1, 0)
    assert oracle.twed(a, ta, b, tb, 1.0, 1.0, 2) == config_golden["cfg1"]["value"]
    a32, b32 = (x.astype(np.float32).astype(np.float64) for x in (a, b))
    assert oracle.twed(a32, ta, b32, tb, 1.0, 1.0, 2) == config_golden["cfg1_f32in"]["value"]
    a, ta, b, tb = make_pair(3000, 3, 12)
    assert oracle.twed(a, ta, b, tb, 1.0, 1.0, 2, threads=0) == \
        config_golden["walk_3000_d3_s12"]["value"]
    AA, TAA = make_set(8, 256, 1, 3)
    BB, TBB = make_set(1000, 256, 1, 4)
    for key, want in config_golden["cfg4"]["entries"].items():
        i, j = map(int, key.split(","))
        if i < 8:
            assert oracle.twed(AA[i], TAA[i], BB[j], TBB[j], 1.0, 1.0, 2) == want


def test_oracle_is_not_product():
    """The product package must never import the oracle."""
    import pathlib
    pkg = pathlib.Path(__file__).resolve().parents[1] / "paper_2007_16135_b200"
    for f in pkg.rglob("*.py"):
        text = f.read_text()
        assert "import oracle" not in text and "from oracle" not in text, f


# ---- LCS: the oracle against the reference's values ----
def lcs_golden():
    return json.loads((GOLDEN / "lcs.json").read_text())


def lcs_case(g):
    rng = np.random.default_rng(g["seed"])
    al = np.array(list(g["alphabet"]))
    return "".join(rng.choice(al, size=g["ns"])), "".join(rng.choice(al, size=g["nt"]))


def test_lcs_oracle_matches_reference_goldens():
    from oracle import oracle as orc
    gold = lcs_golden()
    for c in gold["fixed"]:
        assert orc.lcs(c["s"], c["t"]) == c["value"], c
    for g in gold["generated"]:
        s, t = lcs_case(g)
        assert orc.lcs(s, t) == g["value"], g
    # generic hashable symbols share one code table (core.py:152-160, test_band.py:297)
    assert orc.lcs([1, "x", (2, 3), 4], ["x", (2, 3), 9]) == 2


def test_wide_pairs_match_reference(wide_golden, oracle):
    """d >= 5 (reference lp_dist over any m, _kernels.py:24-48): the oracle
    against the reference's own values (tests/golden/gen_wide.py)."""
    n_exact = 0
    for case in wide_golden["pairs"]:
        va, ta, vb, tb = wide_pair_inputs(case)
        got = oracle.twed(va, ta, vb, tb, case["nu"], case["lam"], case["degree"])
        want = float(dec(case["value"]))
        if exact_expected(case["degree"], va.shape[1]):
            assert same_float(got, want), (case["name"], got, want)
            n_exact += 1
        else:
            assert got == pytest.approx(want, rel=1e-12), case["name"]
    assert n_exact >= 60


def test_wide_batches_match_reference(wide_golden, oracle):
    for name, spec in wide_golden["batches"].items():
        la, lb = wide_batch_inputs(spec)
        got = oracle.twed_batch(la, lb, spec["nu"], spec["lam"], spec["degree"],
                                spec["symmetric"])
        want = wide_golden["matrices"][name]
        assert got.shape == want.shape and np.array_equal(got, want), name
