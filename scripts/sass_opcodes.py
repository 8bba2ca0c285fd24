"""SASS opcode summary of the hot kernels (cuobjdump of the built objects).

    python scripts/sass_opcodes.py [out.json]     (default profiles/sass_opcodes.json)

For each kernel: the whole function's opcode counts and those of its steady
state loop (the innermost backward branch whose body holds the most
arithmetic of the kernel's pipe -- FP64 for the pair sweep, FP32 for the fp32
batch), with per-cell figures where the loop's cell count is known.
"""
from __future__ import annotations

import collections
import json
import re
import subprocess
import sys
from pathlib import Path

REPO = Path(__file__).resolve().parents[1]
OBJ = REPO / "build" / "obj"

KERNELS = {
    # name: (object, mangled-name regex, arithmetic regex, cells per loop iteration)
    "wave_kernel cfg3 (d=3, fp64, k6w12, degree 2, nu=1)": (
        "wave_dd_d3.o", r"wave_kernelILi3ELi6ELi1ELi2ELb0ELb1ELi12ELi1Edd", r"\bD(ADD|MUL|FMA)\b", 12),
    "wave_kernel d=1 fp64 (k6w12)": (
        "wave_dd_d1.o", r"wave_kernelILi1ELi6ELi1ELi2ELb0ELb1ELi12ELi1Edd", r"\bD(ADD|MUL|FMA)\b", 12),
    "batch_kernel cfg5 (d=2, fp32, K=8, 16 lanes per series)": (
        "batch_ff_d2.o", r"batch_kernelILi2ELi8ELi16ELi2ELb0ELb1ELi4Eff", r"\bF(ADD|MUL|FMA)\b", None),
    "prepare_kernel (fp64)": ("twb_api.o", r"prepare_kernelIdddE", r"\bD(ADD|MUL|FMA)\b", None),
    "lcs_kernel": ("twb_lcs.o", r"lcs_kernel", r"\b(IADD3|LOP3)\b", None),
}


def functions(obj: Path) -> dict[str, list[tuple[int, str]]]:
    text = subprocess.run(["cuobjdump", "-sass", str(obj)], capture_output=True, text=True,
                          check=True).stdout
    out, cur = {}, None
    for line in text.split("\n"):
        m = re.match(r"\s*Function : (\S+)", line)
        if m:
            cur = m.group(1)
            out[cur] = []
            continue
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
        if m and cur:
            out[cur].append((int(m.group(1), 16), m.group(2)))
    return out


def opcode(ins: str) -> str:
    return re.sub(r"^@!?U?P\w+\s+", "", ins).split()[0]


def hot_loop(ins, arith):
    """The steady-state loop: among the innermost loops (no backward branch
    nested in their body), the densest in arithmetic."""
    loops = []
    for a, s in ins:
        if "BRA" not in s:
            continue
        t = re.search(r"0x([0-9a-f]+)", s.split("BRA", 1)[1])
        if t and int(t.group(1), 16) < a:
            loops.append((int(t.group(1), 16), a))
    inner = [(lo, hi) for lo, hi in loops
             if not any(lo <= l2 and h2 < hi and (l2, h2) != (lo, hi) for l2, h2 in loops)]
    cand = []
    for lo, hi in inner:
        body = [x for x in ins if lo <= x[0] <= hi]
        n = sum(1 for _, x in body if re.search(arith, x))
        if n:
            cand.append((n, body))
    if not cand:
        return []
    # the steady state: the densest of the loops carrying at least half the
    # largest loop's arithmetic (the pipeline fill is a bigger, sparser loop)
    top = max(n for n, _ in cand)
    return max(((n / len(b), b) for n, b in cand if n >= top / 2), key=lambda t: t[0])[1]


def main():
    dst = Path(sys.argv[1]) if len(sys.argv) > 1 else REPO / "profiles" / "sass_opcodes.json"
    report = {}
    cache = {}
    for name, (obj, pat, arith, cells) in KERNELS.items():
        if obj not in cache:
            cache[obj] = functions(OBJ / obj)
        fns = [f for f in cache[obj] if re.search(pat, f)]
        if not fns:
            report[name] = {"error": f"no function matching {pat} in {obj}"}
            continue
        ins = cache[obj][fns[0]]
        whole = collections.Counter(opcode(s) for _, s in ins)
        loop = hot_loop(ins, arith)
        lc = collections.Counter(opcode(s) for _, s in loop)
        entry = {
            "function": fns[0], "object": obj, "instructions": len(ins),
            "tma_bulk_or_async": {k: v for k, v in whole.items()
                                  if re.match(r"(UBLKCP|UTMALDG|UTMASTG|LDGSTS|SYNCS)", k)},
            "steady_loop": {"instructions": len(loop),
                            "opcodes": dict(lc.most_common())},
        }
        if cells:
            entry["steady_loop"]["cells_per_iteration"] = cells
            entry["steady_loop"]["per_cell"] = {k: round(v / cells, 3) for k, v in lc.most_common()}
            entry["steady_loop"]["instructions_per_cell"] = round(len(loop) / cells, 2)
            entry["steady_loop"]["arith_per_cell"] = round(
                sum(v for k, v in lc.items() if re.search(arith, k)) / cells, 2)
        report[name] = entry
    dst.write_text(json.dumps(report, indent=1) + "\n")
    for name, e in report.items():
        sl = e.get("steady_loop", {})
        print(f"{name}: loop {sl.get('instructions')} instrs, per cell {sl.get('instructions_per_cell')}, "
              f"arith/cell {sl.get('arith_per_cell')}, bulk/async {e.get('tma_bulk_or_async')}")


if __name__ == "__main__":
    main()
