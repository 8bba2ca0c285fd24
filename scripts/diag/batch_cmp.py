"""Compare batch matrices of two library builds (TWB_LIBRARY_B) on short series."""
import os
import subprocess
import sys
from pathlib import Path

import numpy as np

REPO = Path(__file__).resolve().parents[2]
if len(sys.argv) > 1 and sys.argv[1] == "run":
    sys.path.insert(0, str(REPO))
    import paper_2007_16135_b200 as twb
    from paper_2007_16135_b200.workloads import make_set
    res = {}
    for d in (1, 2, 3, 5, 8, 28):
        for n in (16, 28, 32):
            S, T = make_set(150, n, d, d * 100 + n)
            for tri in (True, False):
                res[f"{d}_{n}_{tri}"] = twb.twed_batch(S, T, None, None, 1.0, 1.0, 2, tri)
    np.savez(sys.argv[2], **res)
    sys.exit(0)
out = REPO / "gpurun_out"
env = dict(os.environ)
subprocess.run([sys.executable, __file__, "run", str(out / "cmp_a.npz")], check=True, env=env)
env["TWB_LIBRARY"] = os.environ["TWB_LIBRARY_B"]
subprocess.run([sys.executable, __file__, "run", str(out / "cmp_b.npz")], check=True, env=env)
a, b = np.load(out / "cmp_a.npz"), np.load(out / "cmp_b.npz")
for k in a.files:
    eq = np.array_equal(a[k], b[k])
    print(k, "equal" if eq else f"DIFF max {np.abs(a[k]-b[k]).max():.4g} first {np.argwhere(a[k] != b[k])[:3].tolist()}")
