"""pytest plugin: run the reference package's own test-suite with its band
solvers swapped for the B200 kernels (paper_2007_16135_b200.seam, the S2 seam
of SURVEY.md §8(b)). Used by scripts/run_reference_suite.sh; not collected by
the repo's own tests.

    PYTHONPATH=scripts:baseline/_ref:. python -m pytest -p ref_seam_plugin <reference tests>
"""

import pytest

_handle = None


def pytest_configure(config):
    global _handle
    import twedband

    from paper_2007_16135_b200 import seam

    _handle = seam.install(twedband)
    config.addinivalue_line("markers", "gpu_seam: run against libtwb200")


def pytest_terminal_summary(terminalreporter):
    calls = _handle.calls if _handle is not None else 0
    terminalreporter.write_line(
        f"[ref_seam_plugin] twedband._kernels.twed_band_serial/_parallel -> libtwb200: "
        f"{calls} GPU band solves")
