"""Race hunt: results of the pair sweep under a library variant across
configurations, against the default build's value (diagnostics)."""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import torch  # noqa: E402

import numpy as np  # noqa: E402
import paper_2007_16135_b200 as twb  # noqa: E402
from paper_2007_16135_b200.workloads import make_pair  # noqa: E402

dev = torch.device("cuda:0")
for n, d in ((300_000, 3), (100_000, 3), (300_000, 1), (60_000, 3)):
    a, ta, b, tb = (torch.from_numpy(np.ascontiguousarray(x)).to(dev) for x in make_pair(n, d, 2))
    for cfg in ("", "k8w8", "k6w12", "k4w12"):
        for ws in ("0", "4", "8"):
            if cfg:
                os.environ["TWB_WAVE_CFG"] = cfg
            else:
                os.environ.pop("TWB_WAVE_CFG", None)
            os.environ["TWB_WAVE_WS"] = ws
            vals = set()
            for _ in range(3):
                vals.add(twb.twed_dev(a, ta, b, tb, nu=1.0, lamb=1.0, degree=2).item())
            print(n, d, cfg or "default", "ws", ws, sorted(vals), flush=True)
