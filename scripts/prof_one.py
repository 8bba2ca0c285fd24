"""One call of a workload's hot kernel, for ncu captures (not a bench number).

    python scripts/prof_one.py cfg3|cfg3_f32|cfg2|cfg5 [--n N]
"""
import argparse
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

import paper_2007_16135_b200 as twb  # noqa: E402
from paper_2007_16135_b200.workloads import CONFIGS, make_pair, make_set  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("workload")
ap.add_argument("--n", type=int, default=0)
ap.add_argument("--count", type=int, default=0)
args = ap.parse_args()
cfg = CONFIGS[args.workload]
dev = torch.device("cuda", 0)
if cfg["kind"] == "pair":
    n = args.n or cfg["n"]
    dt = np.float32 if cfg["dtype"] == "f32" else np.float64
    a, ta, b, tb = (torch.from_numpy(np.ascontiguousarray(x.astype(dt))).to(dev)
                    for x in make_pair(n, cfg["d"], cfg["seed"]))
    out = twb.twed_dev(a, ta, b, tb, nu=1.0, lamb=1.0, degree=2)
    torch.cuda.synchronize()
    print(args.workload, n, out.item())
else:
    N = args.count or cfg["count_a"]
    S, T = make_set(N, cfg["n"], cfg["d"], cfg["seed_a"])
    dt = np.float32 if cfg["dtype"] == "f32" else np.float64
    dS = torch.from_numpy(S.astype(dt).reshape(-1, cfg["d"])).to(dev)
    dT = torch.from_numpy(T.astype(dt).reshape(-1)).to(dev)
    off = np.arange(N + 1, dtype=np.int64) * cfg["n"]
    R = twb.twed_batch_dev(dS, off, dT, nu=1.0, lamb=1.0, degree=2, tri=cfg["tri"])
    torch.cuda.synchronize()
    print(args.workload, N, float(R[0, 1]))
