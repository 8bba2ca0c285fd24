"""Wall time of one pair through the single-kernel and the multi-kernel ring paths."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2007_16135_b200 as twb
from paper_2007_16135_b200.workloads import make_pair
n, d = int(sys.argv[1]), int(sys.argv[2])
a, ta, b, tb = make_pair(n, d, 2)
for dev in (0, [0, 0], [0, 0, 0, 0], 0):
    twb.twed(a[:2000], ta[:2000], b[:2000], tb[:2000], 1.0, 1.0, 2, device=dev)
    t0 = time.perf_counter()
    r = twb.twed(a, ta, b, tb, 1.0, 1.0, 2, device=dev)
    dt = time.perf_counter() - t0
    print(f"n={n} d={d} device={dev}: {dt*1e3:.1f} ms  {n*n/dt/1e9:.1f} GCUPS  result={r!r}", flush=True)
