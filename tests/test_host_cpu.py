"""CPU-only checks of the host side: the C-ABI library loads and exports every
symbol include/twb.h declares, validation mirrors the reference, there is no
CPU fallback, and the batch sharding plan is balanced and exact."""

import re
from pathlib import Path

import numpy as np
import pytest

from conftest import has_cuda

REPO = Path(__file__).resolve().parents[1]


def header_symbols():
    text = (REPO / "include" / "twb.h").read_text()
    return sorted(set(re.findall(r"\b(twb_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_header_symbol():
    import ctypes
    from paper_2007_16135_b200 import _lib
    lib = _lib.load()
    syms = header_symbols()
    assert len(syms) >= 15
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(_lib.exported_symbols())
    assert lib.twb_version() == 200
    assert isinstance(ctypes.CDLL(str(_lib.LIB_PATH)), ctypes.CDLL)


def test_library_is_sm100a_build():
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf",
                          str(REPO / "paper_2007_16135_b200" / "lib" / "libtwb200.so")],
                         capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


@pytest.mark.skipif(has_cuda(), reason="checks the no-device error path")
def test_no_cpu_fallback():
    import paper_2007_16135_b200 as twb
    with pytest.raises(twb.TwbError, match="no CPU fallback"):
        twb.twed([1.0, 2.0], [0.0, 1.0], [1.0], [0.0])
    with pytest.raises(twb.TwbError):
        twb.twed_batch([np.ones(3)], None)


def test_validation_matches_reference_messages():
    import paper_2007_16135_b200 as twb
    from paper_2007_16135_b200 import warpband
    with pytest.raises(ValueError, match="3 timestamps for 2 samples"):
        twb.twed([[1.0], [2.0]], [0.0, 1.0, 2.0], [1.0], [0.0])
    with pytest.raises(ValueError, match="3 dimensions"):
        warpband.twed(np.zeros((2, 2, 2)), [0.0, 1.0], [1.0], [0.0])
    with pytest.raises(ValueError, match="A has d=2, B has d=1"):
        warpband.twed([[1.0, 2.0]], [0.0], [1.0], [0.0])
    with pytest.raises(twb.InvalidInputError, match="strictly increasing"):
        twb.twed([1.0, 2.0], [1.0, 1.0], [1.0], [0.0])
    with pytest.raises(twb.InvalidInputError, match="nu must be >= 0"):
        twb.twed([1.0], [0.0], [1.0], [0.0], nu=-1.0)
    with pytest.raises(twb.InvalidInputError, match="degree must be a positive integer"):
        twb.twed([1.0], [0.0], [1.0], [0.0], degree=1.5)
    with pytest.raises(twb.InvalidInputError, match="same collection"):
        warpband.twed_batch([np.array([1.0])], [np.array([2.0])], symmetric=True)
    with pytest.raises(twb.InvalidInputError, match="workers must be"):
        warpband.twed_batch([np.array([1.0])], workers=0)
    with pytest.raises(TypeError):
        twb.twed([1.0], [0.0], [1.0], [0.0], lamb=0.5, lam=0.25)


def test_timeseries_defaults_and_no_copy():
    from paper_2007_16135_b200 import TimeSeries
    from paper_2007_16135_b200.core import as_series
    s = TimeSeries(np.array([1.0, 2.0, 3.0]))
    assert s.values.shape == (3, 1) and list(s.timestamps) == [0.0, 1.0, 2.0]
    v = np.ascontiguousarray(np.random.default_rng(0).random((1000, 3)))
    t = np.arange(1000, dtype=np.float64)
    assert np.shares_memory(as_series(v, t, "series A").values, v)


def test_row_bounds_balanced():
    from paper_2007_16135_b200.distributed import row_bounds
    for n, w in [(10000, 8), (1000, 3), (7, 4), (5, 8)]:
        for tri in (False, True):
            b = row_bounds(n, w, tri)
            assert b[0][0] == 0 and b[-1][1] == n
            assert all(b[k][1] == b[k + 1][0] for k in range(w - 1))
            if n >= 1000:
                work = [sum((n - i) if tri else 1 for i in range(lo, hi)) for lo, hi in b]
                total = sum(work)
                assert max(work) <= total / w * 1.01 + n


def test_symbols_documented_in_integration():
    text = (REPO / "INTEGRATION.md").read_text()
    for s in ("twb_twed_f64", "twb_twed_batch_f64", "twb_band_solve_f64"):
        assert s in text


def test_stacked_batch_input_validated_in_one_pass():
    """Stacked (N, n[, d]) batch inputs are validated with TimeSeries' rules
    (C:37-62) in one vectorised pass and packed without per-series copies."""
    from paper_2007_16135_b200 import api
    from paper_2007_16135_b200.core import InvalidInputError
    p = api._to_list(np.zeros((5, 7, 2)), None, "series_a", np.float64)
    assert len(p) == 5 and p.d == 2 and p.values.shape == (35, 2)
    assert list(p.off) == [0, 7, 14, 21, 28, 35]
    assert np.array_equal(p.times[:7], np.arange(7.0))
    T = np.tile(np.arange(7.0), (5, 1))
    T[3, 4] = T[3, 3]
    with pytest.raises(InvalidInputError, match="strictly increasing"):
        api._to_list(np.zeros((5, 7)), T, "series_a", np.float64)
    with pytest.raises(ValueError, match="timestamps shape"):
        api._to_list(np.zeros((5, 7)), np.zeros((5, 6)), "series_a", np.float64)
    with pytest.raises(InvalidInputError, match="at least one sample"):
        api._to_list(np.zeros((5, 0, 2)), None, "series_a", np.float64)
