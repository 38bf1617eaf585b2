"""Summarises a warm ncu launch list of whole-network passes
(tools/gpu/pass_ncu.sh): the last pass's kernels with time, DRAM bytes and
tensor-pipe activity.
    python tools/pass_table.py gpurun_out/pass/googlenet_b90.csv [kernels_per_pass]"""
import collections
import csv
import sys

rows, hdr = [], None
for x in csv.reader(open(sys.argv[1])):
    if "Kernel Name" in x:
        hdr = x
        continue
    if hdr and len(x) == len(hdr):
        rows.append(dict(zip(hdr, x)))
by = collections.OrderedDict()
for r in rows:
    by.setdefault(r["ID"], {"name": r["Kernel Name"], "grid": r["Grid Size"]})[r["Metric Name"]] = float(
        r["Metric Value"].replace(",", ""))
ks = list(by.values())
n = int(sys.argv[2]) if len(sys.argv) > 2 else len(ks) // 5
tail = ks[-n:]
tot = sum(k["gpu__time_duration.sum"] for k in tail)
agg = collections.defaultdict(float)
for k in tail:
    t = k["gpu__time_duration.sum"] / 1000
    rb = k.get("dram__bytes_read.sum", 0) + k.get("dram__bytes_write.sum", 0)
    kind = k["name"].split("(")[0].split("::")[-1]
    agg[kind] += t
    print(f"{t:8.1f} us {t / tot * 1e5:5.1f}% dram {rb / 1e6:7.1f} MB {rb / (t * 1e-6) / 1e9:6.0f} GB/s "
          f"tensor {k.get('sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active', 0):5.1f}% "
          f"{k['grid']:>14} {k['name'][:60]}")
print(f"kernels {len(tail)} of {len(ks)}; sum {tot / 1000:.1f} us;", {k: round(v, 1) for k, v in agg.items()})
