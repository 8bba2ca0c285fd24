"""LCS kernel timings (twb_lcs_i32, CUDA events around the sweep) at several sizes."""
import sys, time
from pathlib import Path
import numpy as np
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2007_16135_b200 import _lib
from paper_2007_16135_b200.api import lcs_codes
lib = _lib.load()
lib.twb_set_kernel_timing(1)
rng = np.random.default_rng(1)
for n, A in ((100_000, 4), (1_000_000, 4), (1_000_000, 26), (4_000_000, 4)):
    a = rng.integers(0, A, n).astype(np.int64)
    b = rng.integers(0, A, n).astype(np.int64)
    lcs_codes(a[:1000], b[:1000])
    ks = []
    for _ in range(3):
        t0 = time.perf_counter()
        r = lcs_codes(a, b)
        wall = time.perf_counter() - t0
        ks.append(lib.twb_last_kernel_ms())
    k = min(ks)
    print(f"lcs n={n} A={A}: kernel {k:.2f} ms = {n*n/(k*1e-3)/1e9:.0f} GCUPS; wall {wall*1e3:.1f} ms; lcs={r}", flush=True)
