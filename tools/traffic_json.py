"""Per-step DRAM traffic of the dominant kernels from an ncu --metrics
dram__bytes_read.sum,dram__bytes_write.sum --csv launch list (one bench step):
python tools/traffic_json.py launches.csv steps > profiles/traffic_configN.json"""
import csv
import json
import sys
from collections import defaultdict

rows = [r for r in csv.reader(open(sys.argv[1])) if r]
steps = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
hdr = next(r for r in rows if r[0] == "ID")
agg = defaultdict(lambda: {"launches": set(), "bytes": 0.0})
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "KB": 1e3, "MB": 1e6, "GB": 1e9}
for r in rows[rows.index(hdr) + 1:]:
    d = dict(zip(hdr, r))
    if d.get("Metric Name") not in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        continue
    name = d["Kernel Name"].split("(")[0].replace("void ", "").replace("mcf::", "")
    key = "combine" if name.startswith("k_diag_unit") else name.split("<")[0]
    agg[key]["launches"].add(d["ID"])
    agg[key]["bytes"] += float(d["Metric Value"].replace(",", "")) * scale.get(d["Metric Unit"], 1)
out = {k: {"dram_bytes_per_step": v["bytes"] / steps, "launches_per_step": len(v["launches"]) / steps,
           "dram_bytes_per_launch": v["bytes"] / max(1, len(v["launches"]))} for k, v in agg.items()}
print(json.dumps(out, indent=1))
