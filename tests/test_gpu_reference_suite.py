"""The reference's OWN test-suites against the B200 kernels (needs the
reference staged in baseline/ by scripts/stage_reference.sh; skipped without).

1. pkg/tests + pkg/bindings/tests with the S2 kernel seam swapped
   (twedband._kernels.twed_band_serial/_parallel and lcs_band_solve ->
   libtwb200, paper_2007_16135_b200.seam): every reference caller runs on the GPU
   and the suite's bit-equality assertions against its own quadratic oracle
   and exhaustive-path oracle must hold.
2. pkg/bindings/tests with ``warpband`` = paper_2007_16135_b200.warpband (the S1
   drop-in), ``twedband`` = the unmodified reference on the CPU.
"""

import os
import subprocess
import sys

import pytest

from conftest import REPO, has_cuda

SUITE = REPO / "baseline" / "_ref_suite"
REF = REPO / "baseline" / "_ref"

pytestmark = [
    pytest.mark.gpu,
    pytest.mark.skipif(not has_cuda(), reason="needs a CUDA device"),
    pytest.mark.skipif(not (SUITE.is_dir() and (REF / "twedband").is_dir()),
                       reason="reference not staged (scripts/stage_reference.sh)"),
]

# matplotlib is not in the image: the two figure tests cannot run anywhere here
DESELECT = "not test_plot_renders_heatmap and not test_out_writes_csv_and_figures"


def _run(plugin, paths):
    env = dict(os.environ, NUMBA_CACHE_DIR="/tmp/twb_numba_cache",
               PYTHONPATH=os.pathsep.join([str(REPO / "scripts"), str(REF), str(REPO)]))
    cmd = [sys.executable, "-m", "pytest", "-q", "-p", plugin, "-p", "no:cacheprovider",
           "-k", DESELECT, *[str(p) for p in paths]]
    out = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=1500,
                         cwd=str(REPO))
    return out


def test_reference_suite_through_the_kernel_seam():
    out = _run("ref_seam_plugin", [SUITE / "tests", SUITE / "bindings" / "tests"])
    tail = out.stdout[-4000:]
    assert out.returncode == 0, tail + out.stderr[-2000:]
    assert " passed" in tail and "failed" not in tail, tail
    assert "GPU band solves" in tail, tail
    solves = int(tail.split("libtwb200: ")[1].split()[0])
    assert solves > 500, tail


def test_reference_bindings_tests_on_the_dropin_module():
    out = _run("warpband_alias_plugin", [SUITE / "bindings" / "tests"])
    tail = out.stdout[-4000:]
    assert out.returncode == 0, tail + out.stderr[-2000:]
    assert "paper_2007_16135_b200.warpband" in tail, tail
    assert " passed" in tail and "failed" not in tail, tail


def test_seam_batch_routing_one_launch():
    """seam.install(batch=True): the reference's twed_batch (E:183-226) runs as
    ONE all-pairs launch; entries and the symmetric layout equal the
    reference's own CPU batch bit for bit (fp64), ragged lists included."""
    code = r'''
import sys, numpy as np
import twedband as tb
from paper_2007_16135_b200 import seam, _lib
rng = np.random.default_rng(5)
series = [tb.TimeSeries(np.cumsum(rng.standard_normal((int(n), 2)), axis=0),
                        np.cumsum(rng.uniform(0.1, 2.0, int(n))))
          for n in rng.integers(1, 200, 40)]
other = [tb.TimeSeries(np.cumsum(rng.standard_normal((int(n), 2)), axis=0))
         for n in rng.integers(1, 300, 17)]
params = tb.TwedParams(0.5, 0.25, 2)
want_sym = tb.twed_batch(tb.BatchSpec(series, series, params, symmetric=True, workers=4)).entries
want_ab = tb.twed_batch(tb.BatchSpec(series, other, params, workers=4)).entries
h = seam.install(tb, batch=True)
_lib.take_launch_count()
got_sym = tb.twed_batch(tb.BatchSpec(series, series, params, symmetric=True, workers=4))
n_launch = _lib.take_launch_count()
got_ab = tb.engine.twed_batch(tb.BatchSpec(series, other, params, workers=4)).entries
h.restore()
assert got_sym.symmetric and np.array_equal(got_sym.entries, want_sym)
assert np.array_equal(got_ab, want_ab)
assert h.calls == 2 and n_launch <= 4, (h.calls, n_launch)
print("OK", n_launch)
'''
    env = dict(os.environ, NUMBA_CACHE_DIR="/tmp/twb_numba_cache",
               PYTHONPATH=os.pathsep.join([str(REF), str(REPO)]))
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                         timeout=600, cwd=str(REPO))
    assert out.returncode == 0 and "OK" in out.stdout, out.stdout[-2000:] + out.stderr[-3000:]
