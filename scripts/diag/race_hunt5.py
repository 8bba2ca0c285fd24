"""The configurations that raced before the staging wait (diagnostics):
20 sweeps each, distinct results printed. TWB_LIBRARY picks the build."""
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
cases = ((300_000, 3, "k8w8", "8"), (300_000, 3, "", "0"), (60_000, 3, "k8w8", "8"), (100_000, 3, "k8w8", "8"),
         (20_000, 3, "k4w12", "12"), (20_000, 3, "k8w8", "8"), (20_000, 2, "k8w8", "8"), (150_000, 2, "k4w12", "12"))
for n, d, cfg, ws in cases:
    a, ta, b, tb = (torch.from_numpy(np.ascontiguousarray(x)).to(dev) for x in make_pair(n, d, 2))
    if cfg:
        os.environ["TWB_WAVE_CFG"] = cfg
    else:
        os.environ.pop("TWB_WAVE_CFG", None)
    os.environ["TWB_WAVE_WS"] = ws
    vals = [twb.twed_dev(a, ta, b, tb, nu=1.0, lamb=1.0, degree=2).item() for _ in range(20)]
    u = sorted(set(vals))
    bad += len(u) > 1
    print("INCONSISTENT" if len(u) > 1 else "ok", n, d, cfg or "default", ws, u, flush=True)
print("inconsistent cases:", bad, flush=True)
