"""pytest plugin: run the reference bindings' own tests
(pkg/bindings/tests/test_bindings.py) against this repo's drop-in module:
``import warpband`` resolves to ``paper_2007_16135_b200.warpband`` (the B200
kernels), while ``twedband`` stays the unmodified reference (CPU), so every
equality in those tests compares the GPU result with the reference's own.

    PYTHONPATH=scripts:baseline/_ref:. python -m pytest -p warpband_alias_plugin \
        baseline/_ref_suite/bindings/tests
"""

import sys


def pytest_configure(config):
    from paper_2007_16135_b200 import warpband

    sys.modules["warpband"] = warpband


def pytest_terminal_summary(terminalreporter):
    mod = sys.modules.get("warpband")
    terminalreporter.write_line(f"[warpband_alias_plugin] warpband -> {getattr(mod, '__name__', mod)}")
