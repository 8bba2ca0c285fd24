"""cfg5 / cfg4 end to end through twed_batch (numpy in, numpy out), median of
5 calls, and the split: kernel-resident batch vs copy-out (diagnostics)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import numpy as np  # noqa: E402

import paper_2007_16135_b200 as twb  # noqa: E402
from paper_2007_16135_b200.workloads import make_set  # noqa: E402

S, TS = make_set(10000, 128, 2, 5)
S32, TS32 = S.astype(np.float32), TS.astype(np.float32)
AA, TAA = make_set(1000, 256, 1, 3)
BB, TBB = make_set(1000, 256, 1, 4)
for name, call in (("cfg5", lambda: twb.twed_batch(S32, TS32, None, None, 1.0, 1.0, 2, True, dtype=np.float32)),
                   ("cfg4", lambda: twb.twed_batch(AA, TAA, BB, TBB, 1.0, 1.0, 2, False))):
    call()
    ts = []
    for _ in range(5):
        t0 = time.perf_counter()
        R = call()
        ts.append(time.perf_counter() - t0)
    print(name, "e2e ms median %.1f min %.1f" % (1e3 * np.median(ts), 1e3 * min(ts)), R.shape, flush=True)
