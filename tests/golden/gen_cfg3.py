"""cfg3 goldens (n=1,000,000, d=3 pair) from the pinned CPU oracle.

The reference's own band takes ~2 h per value on 8 cores, so
these come from oracle/twed_oracle.c's bit-identical tiled schedule
(orc_band_tiled), which reproduces every reference golden bit for bit
(tests/test_oracle_golden.py). Run in the build container:

    python tests/golden/gen_cfg3.py [threads]
"""

import json
import sys
import time
from pathlib import Path

import numpy as np

REPO = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(REPO))

from oracle import oracle as o  # noqa: E402
from paper_2007_16135_b200.workloads import make_pair  # noqa: E402

OUT = Path(__file__).resolve().parent / "cfg3.json"


def main():
    threads = int(sys.argv[1]) if len(sys.argv) > 1 else 0
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 1_000_000
    res = json.loads(OUT.read_text()) if OUT.exists() else {}
    a, ta, b, tb = make_pair(n, 3, 2)
    key = f"cfg3_n{n}"
    if key not in res:
        t0 = time.time()
        v = o.twed_tiled(a, ta, b, tb, 1.0, 1.0, 2, threads=threads, tile=512)
        res[key] = {"seed": 2, "n": n, "d": 3, "value": v, "seconds": time.time() - t0,
                    "how": "oracle.orc_band_tiled (bit-identical schedule of the reference band)"}
        OUT.write_text(json.dumps(res, indent=1))
        print(key, v, flush=True)
    key32 = key + "_f32in"
    if key32 not in res:
        a32, b32 = (x.astype(np.float32).astype(np.float64) for x in (a, b))
        t0 = time.time()
        v = o.twed_tiled(a32, ta, b32, tb, 1.0, 1.0, 2, threads=threads, tile=512)
        res[key32] = {"value": v, "seconds": time.time() - t0,
                      "how": "fp64 oracle on fp32-rounded inputs"}
        OUT.write_text(json.dumps(res, indent=1))
        print(key32, v, flush=True)


if __name__ == "__main__":
    main()
