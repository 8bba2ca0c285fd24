"""profiles/ncu_summary.json from an ncu DRAM-bytes capture of the cfg3 wave kernel
(gpu_run.sh ncu_wave: dram__bytes_read.sum + dram__bytes_write.sum, one launch).

    python scripts/make_ncu_summary.py gpurun_out/<tag>_wave_cfg3_dram.csv
"""
import csv
import json
import sys
from pathlib import Path

src = Path(sys.argv[1])
rows = [r for r in csv.reader(open(src)) if len(r) > 10 and r[0] != "ID"]
vals = {r[12]: float(r[14].replace(",", "")) for r in rows}
out = Path(__file__).resolve().parents[1] / "profiles" / "ncu_summary.json"
summary = json.loads(out.read_text()) if out.exists() else {}
summary["cfg3"] = {
    "kernel": rows[0][4],
    "grid": rows[0][8],
    "dram_bytes_read": vals["dram__bytes_read.sum"],
    "dram_bytes_write": vals["dram__bytes_write.sum"],
    "dram_bytes": vals["dram__bytes_read.sum"] + vals["dram__bytes_write.sum"],
    "duration_ns_under_ncu": vals.get("gpu__time_duration.sum"),
    "source": src.name,
    "note": ("per launch (one launch = one 1M x 1M pair). Writes are the stripes' bottom "
             "rows (z, d: 16 B per column per stripe) evicted from L2; the next stripe "
             "reads them back mostly from L2."),
}
out.write_text(json.dumps(summary, indent=1) + "\n")
print(json.dumps(summary["cfg3"], indent=1))
