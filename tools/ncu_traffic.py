"""DRAM traffic per launch of one kernel from an ncu --set full report
(used for bench.py's roofline.traffic).
usage: python tools/ncu_traffic.py report.ncu-rep kernel_regex source_note > out.json"""
import csv
import io
import json
import re
import subprocess
import sys

rep, pat, note = sys.argv[1], sys.argv[2], sys.argv[3]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, unit = rows[0], rows[1]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "nsecond": 1e-9, "us": 1e-6,
         "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3}
def val(r, k):
    i = hdr.index(k)
    return float(r[i].replace(",", "")) * scale[unit[i]]
per = []
for r in rows[2:]:
    if not re.search(pat, r[hdr.index("Kernel Name")]):
        continue
    per.append({"time_s": val(r, "gpu__time_duration.sum"),
                "dram_bytes": val(r, "dram__bytes_read.sum") + val(r, "dram__bytes_write.sum"),
                "grid": r[hdr.index("launch__grid_size")], "block": r[hdr.index("launch__block_size")]})
tot_b = sum(p["dram_bytes"] for p in per)
out = {"kernel": pat, "source": note, "launches": len(per), "dram_bytes_total": tot_b,
       "time_s_total": sum(p["time_s"] for p in per), "dram_bytes_per_launch": tot_b / max(1, len(per)),
       "per_launch": per}
print(json.dumps(out, indent=1))
