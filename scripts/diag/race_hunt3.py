"""Stress of the headline configuration (k6w12, rows in shared memory,
pipelined fill): repeated sweeps over sizes and stripe heights; any
disagreement between repetitions is printed (diagnostics)."""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2007_16135_b200 as twb  # noqa: E402
from paper_2007_16135_b200.workloads import make_pair  # noqa: E402

dev = torch.device("cuda:0")
cfg = os.environ.get("CFG", "k6w12")
os.environ["TWB_WAVE_CFG"] = cfg
bad = 0
for n, d in ((20_000, 3), (60_000, 3), (60_000, 2), (150_000, 3), (300_000, 2)):
    a, ta, b, tb = (torch.from_numpy(np.ascontiguousarray(x)).to(dev) for x in make_pair(n, d, 7))
    for ws in ("4", "8", "12"):
        os.environ["TWB_WAVE_WS"] = ws
        vals = [twb.twed_dev(a, ta, b, tb, nu=1.0, lamb=1.0, degree=2).item() for _ in range(8)]
        u = sorted(set(vals))
        bad += len(u) > 1
        print(cfg, n, d, "ws", ws, "distinct", len(u), u if len(u) > 1 else u[0], flush=True)
print("inconsistent cases:", bad)
