"""Batch of mid-length series (rows > 256 samples: per-pair wavefront solves)."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import numpy as np
import paper_2007_16135_b200 as twb
rng = np.random.default_rng(3)
for N, n, tri in ((100, 1000, True), (64, 3000, False)):
    S = [np.cumsum(rng.standard_normal((n, 1)), axis=0) for _ in range(N)]
    twb.twed_batch(S[:3], None, None, None, 1.0, 1.0, 2, tri)
    t0 = time.perf_counter()
    R = twb.twed_batch(S, None, None, None, 1.0, 1.0, 2, tri)
    dt = time.perf_counter() - t0
    pairs = N * (N + 1) // 2 if tri else N * N
    ref = twb.twed(S[3], np.arange(n, dtype=float), S[7], np.arange(n, dtype=float), 1.0, 1.0, 2)
    assert R[3, 7] == ref and R[7, 3] == ref
    print(f"N={N} n={n} tri={tri}: {dt*1e3:.0f} ms, {pairs/dt:.0f} pairs/s, {pairs*n*n/dt/1e9:.1f} GCUPS", flush=True)
