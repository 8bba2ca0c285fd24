"""Summarise an ncu --set full report (.ncu-rep) into JSON: speed-of-light,
issue/IPC, FP64/FP32 pipe utilisation, DRAM bytes, registers/occupancy and the
top stall reasons (from the source page). Runs here (no GPU needed).

    python scripts/summarize_ncu.py gpurun_out/x.ncu-rep [--out profiles/x.json]
"""
import argparse
import csv
import io
import json
import subprocess
from collections import Counter

NCU = "/usr/local/cuda/bin/ncu"

WANT = {
    "gpu__time_duration.sum": "duration_ns",
    "dram__bytes_read.sum": "dram_bytes_read",
    "dram__bytes_write.sum": "dram_bytes_write",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
    "sm__inst_executed.avg.per_cycle_active": "ipc_active",
    "sm__instruction_throughput.avg.pct_of_peak_sustained_active": "issue_pct",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "fp64_pipe_pct",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active": "fp64_inst_pct",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active": "fma_pipe_pct",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active": "alu_pipe_pct",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active": "xu_pipe_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "achieved_occupancy_pct",
    "launch__registers_per_thread": "registers_per_thread",
    "launch__grid_size": "grid_size",
    "launch__block_size": "block_size",
    "smsp__inst_executed.sum": "warp_instructions",
}


def raw(path):
    out = subprocess.run([NCU, "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    head, units = rows[0], rows[1]
    res = []
    unit_of = dict(zip(head, units))
    scale = {"nsecond": 1.0, "usecond": 1e3, "msecond": 1e6, "second": 1e9, "ns": 1.0,
             "us": 1e3, "ms": 1e6, "s": 1e9,
             "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    for r in rows[2:]:
        d = dict(zip(head, r))
        entry = {"kernel": d.get("Kernel Name", "")[:160]}
        for k, name in WANT.items():
            if k in d and d[k] not in ("", "n/a"):
                try:
                    v = float(d[k].replace(",", ""))
                except ValueError:
                    entry[name] = d[k]
                    continue
                entry[name] = v * scale.get(unit_of.get(k, ""), 1.0)
        res.append(entry)
    return res


def stalls(path):
    out = subprocess.run([NCU, "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        return {}
    head = rows[1]
    tot = Counter()
    for r in rows[2:]:
        if len(r) != len(head):
            continue
        d = dict(zip(head, r))
        for c in head:
            if c.startswith("stall_") and "Not Issued" not in c:
                try:
                    tot[c[6:]] += int(d[c] or 0)
                except ValueError:
                    pass
    n = sum(tot.values()) or 1
    return {k: round(100.0 * v / n, 1) for k, v in tot.most_common(8)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--out")
    args = ap.parse_args()
    summary = {"report": args.rep, "kernels": raw(args.rep), "stall_pct_of_samples": stalls(args.rep)}
    for k in summary["kernels"]:
        if "dram_bytes_read" in k and "dram_bytes_write" in k:
            k["dram_bytes"] = k["dram_bytes_read"] + k["dram_bytes_write"]
    text = json.dumps(summary, indent=1)
    if args.out:
        open(args.out, "w").write(text + "\n")
    print(text)


if __name__ == "__main__":
    main()
