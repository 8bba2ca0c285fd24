"""Quick kernel timings for tuning (device-resident inputs, CUDA events inside
libtwb200). Not a bench number: no L2 flush, no clocks.

    python scripts/tune.py pair  N D dtype [WS ...]     # wave kernel, GCUPS per TWB_WAVE_WS
    python scripts/tune.py batch N n D dtype tri        # batch kernel
"""
import os
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_2007_16135_b200 as twb  # noqa: E402
from paper_2007_16135_b200 import _lib  # noqa: E402
from paper_2007_16135_b200.workloads import make_pair, make_set  # noqa: E402

lib = _lib.load()
lib.twb_set_kernel_timing(1)
dev = torch.device("cuda", 0)
kind = sys.argv[1]
if kind == "pair":
    n, d, dt = int(sys.argv[2]), int(sys.argv[3]), sys.argv[4]
    wss = sys.argv[5:] or ["0"]
    npdt = np.float32 if dt == "f32" else np.float64
    a, ta, b, tb = (torch.from_numpy(np.ascontiguousarray(x.astype(npdt))).to(dev)
                    for x in make_pair(n, d, 2))
    for ws in wss:
        os.environ["TWB_WAVE_WS"] = ws
        out = twb.twed_dev(a, ta, b, tb, nu=1.0, lamb=1.0, degree=2)
        lib.twb_last_kernel_ms()
        ks = []
        reps = 3 if n * n * d > 1e11 else 10
        for _ in range(reps):
            twb.twed_dev(a, ta, b, tb, nu=1.0, lamb=1.0, degree=2, out=out)
            ks.append(lib.twb_last_kernel_ms())
        k = min(ks)
        print(f"pair n={n} d={d} {dt} ws={ws}: {k:.3f} ms  {n*n/k/1e6:.1f} GCUPS  "
              f"result={out.item()!r}", flush=True)
elif kind == "pair2":  # pair2 nA nB d dtype [reps]: rows nA (TWB_NO_SWAP set)
    os.environ["TWB_NO_SWAP"] = "1"
    na, nb, d, dt = int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]), sys.argv[5]
    npdt = np.float32 if dt == "f32" else np.float64
    rng = np.random.default_rng(3)
    a = torch.from_numpy(np.cumsum(rng.standard_normal((na, d)), 0).astype(npdt)).to(dev)
    b = torch.from_numpy(np.cumsum(rng.standard_normal((nb, d)), 0).astype(npdt)).to(dev)
    ta = torch.arange(na, dtype=a.dtype, device=dev)
    tb = torch.arange(nb, dtype=a.dtype, device=dev)
    out = twb.twed_dev(a, ta, b, tb, nu=1.0, lamb=1.0, degree=2)
    lib.twb_last_kernel_ms()
    ks = []
    for _ in range(2):
        twb.twed_dev(a, ta, b, tb, nu=1.0, lamb=1.0, degree=2, out=out)
        ks.append(lib.twb_last_kernel_ms())
    k = min(ks)
    print(f"pair2 nA={na} nB={nb} d={d} {dt} cfg={os.environ.get('TWB_WAVE_CFG')}: {k:.3f} ms "
          f"{na*nb/k/1e6:.2f} GCUPS  {k*1e-3*1.965e9/nb:.0f} cycles/column", flush=True)
else:
    N, n, d, dt, tri = int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]), sys.argv[5], \
        sys.argv[6] == "1"
    npdt = np.float32 if dt == "f32" else np.float64
    S, T = make_set(N, n, d, 5)
    dS = torch.from_numpy(S.astype(npdt).reshape(-1, d)).to(dev)
    dT = torch.from_numpy(T.astype(npdt).reshape(-1)).to(dev)
    off = np.arange(N + 1, dtype=np.int64) * n
    R = twb.twed_batch_dev(dS, off, dT, nu=1.0, lamb=1.0, degree=2, tri=tri)
    lib.twb_last_kernel_ms()
    ks = []
    for _ in range(3):
        twb.twed_batch_dev(dS, off, dT, nu=1.0, lamb=1.0, degree=2, tri=tri, out=R)
        ks.append(lib.twb_last_kernel_ms())
    k = min(ks)
    pairs = N * (N + 1) // 2 if tri else N * N
    print(f"batch N={N} n={n} d={d} {dt} tri={tri}: {k:.3f} ms  {pairs/k*1e3/1e6:.2f} Mpairs/s  "
          f"{pairs*n*n/k/1e6:.1f} GCUPS", flush=True)
