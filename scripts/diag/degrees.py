import sys, time
sys.path.insert(0, '/root/repo')
import numpy as np
import paper_2007_16135_b200 as twb
from paper_2007_16135_b200.workloads import make_pair
a, ta, b, tb = make_pair(100000, 2, 3)
for deg in (2, 1, 3, 4):
    twb.twed(a[:1000], ta[:1000], b[:1000], tb[:1000], 1.0, 1.0, deg)
    t0 = time.perf_counter(); r = twb.twed(a, ta, b, tb, 1.0, 1.0, deg); dt = time.perf_counter() - t0
    print(f"degree {deg}: {dt*1e3:.1f} ms {1e10/dt/1e9:.1f} GCUPS r={r!r}")
