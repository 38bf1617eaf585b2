"""Combine the ncu launch list of tools/traffic_replay.py (dram bytes per
launch) with the executor's algorithmic bytes of the same launches into
profiles/ncu_conv_summary.json."""
import csv
import json
import sys
from collections import defaultdict

csv_path, stats_path = sys.argv[1], sys.argv[2]
out_path = sys.argv[3] if len(sys.argv) > 3 else "profiles/ncu_conv_summary.json"
rows = list(csv.reader(l for l in open(csv_path) if l.startswith('"')))
hdr = rows[0]
ix = {k: hdr.index(k) for k in ("ID", "Kernel Name", "Metric Name", "Metric Unit", "Metric Value")}
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "ns": 1e-3, "usecond": 1, "us": 1, "msecond": 1e3, "ms": 1e3}
per = defaultdict(dict)
for r in rows[1:]:
    v = float(r[ix["Metric Value"]].replace(",", "")) * scale.get(r[ix["Metric Unit"]], 1)
    per[r[ix["ID"]]][r[ix["Metric Name"]]] = v
    per[r[ix["ID"]]]["name"] = r[ix["Kernel Name"]]
conv = [d for d in per.values() if "conv_tc_kernel" in d["name"]]
n = len(conv)
dram = sum(d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0) for d in conv)
us = sum(d.get("gpu__time_duration.sum", 0) for d in conv)
st = json.load(open(stats_path))
c = st["stats"]["conv_tc"]
alg_per = c["bytes"] / c["launches"]
summary = {
    "capture": "ncu --profile-from-start off --clock-control none --metrics gpu__time_duration.sum,"
               "dram__bytes_read.sum,dram__bytes_write.sum over every launch of the config-2 workload replayed "
               "at its capacity rate (tools/traffic_replay.py, tools/traffic_summary.py)",
    "requests": st["requests"], "rate": st["rate"],
    "conv_launches_ncu": n, "conv_launches_accounted": c["launches"],
    "dram_bytes_per_launch": dram / n if n else None,
    "algorithmic_bytes_per_launch": alg_per,
    "dram_over_algorithmic": (dram / n) / alg_per if n else None,
    "conv_us_per_launch_ncu": us / n if n else None,
    "all_kernels": {k: sum(1 for d in per.values() if d["name"] == k) for k in sorted({d["name"] for d in per.values()})},
}
json.dump(summary, open(out_path, "w"), indent=1)
print(json.dumps(summary, indent=1))
