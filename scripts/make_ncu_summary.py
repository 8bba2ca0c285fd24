"""profiles/ncu_summary.json entries from ncu metric captures (gpu_run.sh
ncu_dram: dram__bytes_read.sum, dram__bytes_write.sum, gpu__time_duration.sum
of one launch, --csv --log-file).

    python scripts/make_ncu_summary.py cfg3 gpurun_out/<tag>_wave_cfg3_dram.csv
    python scripts/make_ncu_summary.py prepare gpurun_out/<tag>_prepare_cfg3_dram.csv

bench.py reads "cfg3" (the sweep's roofline.traffic) and "prepare" (the
precompute's roofline.traffic).
"""
import csv
import json
import sys
from pathlib import Path

SCALE = {"byte": 1, "kbyte": 1e3, "mbyte": 1e6, "gbyte": 1e9, "tbyte": 1e12,
         "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0,
         "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0}
NOTES = {
    "cfg3": ("per launch (one launch = one 1M x 1M pair). Writes: the round-wrap inbox row and "
             "ring lines evicted from L2; the stripes' bottom rows otherwise stay in L2."),
    "prepare": ("per launch: both cfg3 series (2 x 1M samples, d = 3, fp64) and the input "
                "check; algorithmic 144 MB (read 64 MB, write 80 MB)."),
}


def main():
    key, src = sys.argv[1], Path(sys.argv[2])
    rows = list(csv.reader(open(src)))
    hdr = next(r for r in rows if "Metric Name" in r)
    ih = {h: i for i, h in enumerate(hdr)}
    data = [r for r in rows if len(r) == len(hdr) and r is not hdr and r[ih["Metric Name"]] != "Metric Name"]
    vals = {}
    for r in data:
        unit = r[ih["Metric Unit"]].strip().lower()
        v = float(r[ih["Metric Value"]].replace(",", ""))
        vals[r[ih["Metric Name"]]] = v * SCALE.get(unit, 1.0)
    out = Path(__file__).resolve().parents[1] / "profiles" / "ncu_summary.json"
    summary = json.loads(out.read_text()) if out.exists() else {}
    rd, wr = vals["dram__bytes_read.sum"], vals["dram__bytes_write.sum"]
    summary[key] = {
        "kernel": data[0][ih["Kernel Name"]][:160],
        "grid": data[0][ih["Grid Size"]] if "Grid Size" in ih else None,
        "dram_bytes_read": rd, "dram_bytes_write": wr, "dram_bytes": rd + wr,
        "duration_s_under_ncu": vals.get("gpu__time_duration.sum"),
        "source": src.name, "note": NOTES.get(key, ""),
    }
    out.write_text(json.dumps(summary, indent=1) + "\n")
    print(json.dumps(summary[key], indent=1))


if __name__ == "__main__":
    main()
