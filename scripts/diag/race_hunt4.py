"""Repetition hunt over every wavefront configuration and stripe height
(diagnostics): 10 sweeps per case, distinct results printed."""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2007_16135_b200 as twb  # noqa: E402
from paper_2007_16135_b200.workloads import make_pair  # noqa: E402

dev = torch.device("cuda:0")
bad = 0
for n, d in ((20_000, 3), (20_000, 2), (60_000, 3), (150_000, 2)):
    a, ta, b, tb = (torch.from_numpy(np.ascontiguousarray(x)).to(dev) for x in make_pair(n, d, 2))
    for cfg, wss in (("k6w12", ("4", "8", "12")), ("k8w8", ("4", "8")), ("k4w12", ("4", "8", "12"))):
        os.environ["TWB_WAVE_CFG"] = cfg
        for ws in wss:
            os.environ["TWB_WAVE_WS"] = ws
            vals = [twb.twed_dev(a, ta, b, tb, nu=1.0, lamb=1.0, degree=2).item() for _ in range(10)]
            u = sorted(set(vals))
            bad += len(u) > 1
            if len(u) > 1:
                print("INCONSISTENT", cfg, ws, n, d, u, flush=True)
print("inconsistent cases:", bad, flush=True)
