"""Kernel time of the fused pair precompute (bench.py's run_precompute)."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import bench  # noqa: E402

class A:
    pass

print(json.dumps(bench.run_precompute(A(), 0)))
