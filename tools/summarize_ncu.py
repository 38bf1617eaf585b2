"""Summaries of ncu artifacts for profiles/ (run here, on the CPU box).

    python tools/summarize_ncu.py launches gpurun_out/launches_bench.csv profiles/r01/launches_bench_summary.json
    python tools/summarize_ncu.py full gpurun_out/prof_conv.ncu-rep profiles/ncu_conv_summary.json

`launches`: per-kernel launch count, device time and share of the listed
launches (cold-cache, serialised ncu timings: compare shares, not absolutes).
`full`: the headline metrics of every captured launch of a `--set full`
report plus dram_bytes_per_launch (read + write), which bench.py reports as
roofline.traffic.
"""
from __future__ import annotations

import collections
import csv
import io
import json
import subprocess
import sys

FULL_METRICS = [
    "gpu__time_duration.sum",
    "launch__grid_size",
    "launch__block_size",
    "launch__registers_per_thread",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__throughput.avg.pct_of_peak_sustained_active",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
]


def _unit_scale(unit: str) -> float:
    return {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1, "usecond": 1,
            "msecond": 1e3, "nsecond": 1e-3}.get(unit, 1.0)


def launches(src: str, dst: str) -> None:
    txt = open(src).read()
    txt = txt[txt.index('"ID"'):]
    per = collections.OrderedDict()
    for r in csv.DictReader(io.StringIO(txt)):
        d = per.setdefault(r["ID"], {"kernel": r["Kernel Name"].split("(")[0]})
        v = float(r["Metric Value"].replace(",", ""))
        if r["Metric Name"] == "gpu__time_duration.sum":
            d["us"] = v * (1e-3 if r["Metric Unit"] == "ns" else _unit_scale(r["Metric Unit"]))
        elif r["Metric Name"].startswith("dram__bytes"):
            d["dram"] = d.get("dram", 0.0) + v * _unit_scale(r["Metric Unit"])
    agg = collections.defaultdict(lambda: {"launches": 0, "us": 0.0, "dram_bytes": 0.0})
    for d in per.values():
        a = agg[d["kernel"]]
        a["launches"] += 1
        a["us"] += d.get("us", 0.0)
        a["dram_bytes"] += d.get("dram", 0.0)
    tot = sum(a["us"] for a in agg.values())
    out = {"source": src, "launches": len(per), "total_us": round(tot, 1), "kernels": {}}
    for k, a in sorted(agg.items(), key=lambda x: -x[1]["us"]):
        out["kernels"][k] = {"launches": a["launches"], "us": round(a["us"], 1),
                             "share": round(a["us"] / tot, 4) if tot else None,
                             "avg_us": round(a["us"] / a["launches"], 2),
                             "dram_GBps": round(a["dram_bytes"] / (a["us"] * 1e3), 1) if a["us"] else None}
    json.dump(out, open(dst, "w"), indent=1)
    print(json.dumps(out["kernels"], indent=1)[:1500])


def full(rep: str, dst: str) -> None:
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    kernels = []
    for d in data:
        e = {"Kernel Name": d[hdr.index("Kernel Name")], "Grid Size": d[hdr.index("Grid Size")],
             "Block Size": d[hdr.index("Block Size")]}
        for m in FULL_METRICS:
            if m in hdr:
                i = hdr.index(m)
                e[m] = f"{d[i]} {units[i]}".strip()
        kernels.append(e)

    def val(e, m):
        v, _, u = e[m].partition(" ")
        return float(v.replace(",", "")) * _unit_scale(u)

    dram = [val(e, "dram__bytes_read.sum") + val(e, "dram__bytes_write.sum") for e in kernels]
    out = {"capture": f"ncu --set full --clock-control none ({rep})", "kernels": kernels,
           "dram_bytes_per_launch": sum(dram) / len(dram) if dram else None}
    json.dump(out, open(dst, "w"), indent=1)
    print(json.dumps(out, indent=1)[:2500])


if __name__ == "__main__":
    {"launches": launches, "full": full}[sys.argv[1]](sys.argv[2], sys.argv[3])
