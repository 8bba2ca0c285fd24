"""Race hunt 2: k8w8 with 8 active warps, d = 3 (the configuration that
showed a nondeterministic +2432): 10 repetitions per case."""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2007_16135_b200 as twb  # noqa: E402
from paper_2007_16135_b200.workloads import make_pair  # noqa: E402

dev = torch.device("cuda:0")
os.environ["TWB_WAVE_CFG"] = "k8w8"
os.environ["TWB_WAVE_WS"] = "8"
for n, d in ((60_000, 3), (20_000, 3), (60_000, 2), (60_000, 4)):
    a, ta, b, tb = (torch.from_numpy(np.ascontiguousarray(x)).to(dev) for x in make_pair(n, d, 2))
    vals = [twb.twed_dev(a, ta, b, tb, nu=1.0, lamb=1.0, degree=2).item() for _ in range(10)]
    u = sorted(set(vals))
    print(n, d, len(u), "distinct", u, "counts", [vals.count(x) for x in u], flush=True)
