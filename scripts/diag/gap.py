"""Where does the device-resident cfg3 step spend time outside the wave kernel?
Host timestamps around each part of bench.py's step (diagnostic, not a bench)."""
import sys, time
from pathlib import Path
import numpy as np
sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import torch
import paper_2007_16135_b200 as twb
from paper_2007_16135_b200 import _lib
from paper_2007_16135_b200.workloads import make_pair

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
lib = _lib.load()
dev = torch.device("cuda", 0)
a, ta, b, tb = (torch.from_numpy(x).to(dev) for x in make_pair(n, 3, 2))
out = torch.empty(1, dtype=torch.float64, device=dev)
l2 = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)
st = torch.cuda.current_stream(dev)
for timing in (1, 0):
    lib.twb_set_kernel_timing(timing)
    for it in range(4):
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record(st)
        l2.add_(1)
        t1 = time.perf_counter()
        twb.twed_dev(a, ta, b, tb, nu=1.0, lamb=1.0, degree=2, out=out, stream=st)
        t2 = time.perf_counter()
        e1.record(st)
        km = lib.twb_last_kernel_ms() if timing else float("nan")
        torch.cuda.synchronize()
        t3 = time.perf_counter()
        print(f"timing={timing} it={it} step_ev={e0.elapsed_time(e1):9.2f} ms kernel={km:9.2f} "
              f"host: flush {1e3*(t1-t0):7.2f} twed_dev-call {1e3*(t2-t1):9.2f} wait {1e3*(t3-t2):9.2f}",
              flush=True)
