"""One LCS sweep for ncu captures: python scripts/lcs_prof.py N A"""
import sys
from pathlib import Path
import numpy as np
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2007_16135_b200.api import lcs_codes
n, A = int(sys.argv[1]), int(sys.argv[2])
rng = np.random.default_rng(1)
print(lcs_codes(rng.integers(0, A, n), rng.integers(0, A, n)))
