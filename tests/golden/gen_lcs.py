"""Golden LCS lengths computed BY THE REFERENCE (twedband.lcs_band, band.py:185-197,
cross-checked with twedband.lcs_reference, the quadratic table). Run in the build
container (needs /root/reference and numba):

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/nb python tests/golden/gen_lcs.py

Generated strings are re-created by the tests from (seed, alphabet, lengths) with
numpy's default_rng, so only the recipe and the value are stored.
"""
import json
from pathlib import Path

import numpy as np
from twedband import lcs_band, lcs_reference


def make(seed, alphabet, ns, nt):
    rng = np.random.default_rng(seed)
    al = np.array(list(alphabet))
    return "".join(rng.choice(al, size=ns)), "".join(rng.choice(al, size=nt))


def main():
    fixed = [("ABCBDAB", "BDCABA"), ("GATTACA", "GATTACA"), ("", ""), ("", "XYZ"), ("XYZ", ""),
             ("A", "A"), ("A", "B"), ("ACGTACGT", "TGCA"), ("héllo wörld", "hello world"),
             ("x" * 130, "x" * 70 + "y" * 70)]
    out = {"fixed": [], "generated": []}
    for s, t in fixed:
        v = lcs_band(s, t)
        assert v == lcs_reference(s, t)
        out["fixed"].append({"s": s, "t": t, "value": int(v)})
    rng = np.random.default_rng(2007)
    recipes = []
    for k in range(60):  # reference test_band.py:285-289 style, wider
        recipes.append((1000 + k, "ACGT", int(rng.integers(0, 200)), int(rng.integers(0, 200))))
    for k in range(20):
        recipes.append((2000 + k, "ACGTNXYZ01234567"[: int(rng.integers(1, 17))],
                        int(rng.integers(0, 700)), int(rng.integers(0, 700))))
    recipes += [(3001, "ACGT", 2048, 3000), (3002, "AB", 4097, 129), (3003, "ACGT", 63, 5000),
                (3004, "abcdefghijklmnopqrstuvwxyz", 3000, 2500), (3005, "ACGT", 6000, 6000)]
    for seed, al, ns, nt in recipes:
        s, t = make(seed, al, ns, nt)
        v = lcs_band(s, t)
        if ns * nt <= 4_000_000:
            assert v == lcs_reference(s, t)
        out["generated"].append({"seed": seed, "alphabet": al, "ns": ns, "nt": nt,
                                 "value": int(v)})
    path = Path(__file__).resolve().parent / "lcs.json"
    path.write_text(json.dumps(out, indent=0, ensure_ascii=False) + "\n")
    print(f"wrote {path}: {len(out['fixed'])} fixed, {len(out['generated'])} generated")


if __name__ == "__main__":
    main()
