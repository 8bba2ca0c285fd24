"""Repeatability diagnostics of the wavefront (twed through the fused
precompute, and the S2 seam on host-prepared arrays) on multi-round sweeps."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import paper_2007_16135_b200 as twb  # noqa: E402
from oracle import oracle as orc  # noqa: E402
from paper_2007_16135_b200.workloads import make_pair  # noqa: E402

for n, d, seed in ((400000, 1, 11), (400000, 3, 11), (1000000, 1, 2), (250000, 2, 5)):
    a, ta, b, tb = make_pair(n, d, seed)
    vals = [twb.twed(a, ta, b, tb, 1.0, 1.0, 2) for _ in range(5)]
    pa = orc.prepare_series(a, ta, 1.0, 1.0, 2)
    pb = orc.prepare_series(b, tb, 1.0, 1.0, 2)
    seam = [twb.band_solve(pa, pb, 1.0, 2) for _ in range(3)]
    print(n, d, "consistent" if len(set(vals + seam)) == 1 else "INCONSISTENT", vals, seam,
          flush=True)
