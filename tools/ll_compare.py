"""Per-launch comparison of two ncu launch lists of tools/run_layers.py
(BS_CONV_LOG shapes joined to conv launches):
    python tools/ll_compare.py gpurun_out/ll_b90_t0 gpurun_out/ll_b90_t1
"""
import collections
import csv
import io
import re
import sys


def load(stem):
    txt = open(stem + ".csv").read()
    txt = txt[txt.index('"ID"'):]
    L = collections.OrderedDict()
    for r in csv.DictReader(io.StringIO(txt)):
        d = L.setdefault(r["ID"], {"name": r["Kernel Name"], "grid": r["Grid Size"]})
        d[r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
    convs = [l for l in open(stem + ".log") if l.startswith("conv")]
    out, ci = [], 0
    for v in L.values():
        t = v["gpu__time_duration.sum"] / 1000
        dram = (v.get("dram__bytes_read.sum", 0) + v.get("dram__bytes_write.sum", 0)) / 1e6
        if "conv_tc" in v["name"]:
            m = dict(re.findall(r"(\w+)=(\S+)", convs[ci]))
            ci += 1
            fl = 2 * int(m["M"]) * int(m["N"]) * int(m["K"])
            out.append(("conv", f"M={m['M']} N={m['N']} K={m['K']} tma={m.get('tma', '0')} ks={m['ks']}", t, fl, dram))
        else:
            out.append((v["name"].split("(")[0].split("::")[-1][:14], v["grid"], t, 0, dram))
    return out


def main():
    runs = [load(s) for s in sys.argv[1:]]
    tot = [collections.defaultdict(float) for _ in runs]
    for i, rows in enumerate(zip(*runs)):
        line = f"{i:3d} {rows[0][0]:14s} {rows[0][1]:40s}"
        for j, r in enumerate(rows):
            tot[j][r[0]] += r[2]
            tf = r[3] / r[2] / 1e6 if r[3] else 0
            line += f" | {r[2]:7.1f}us {tf:5.0f}TF {r[4]:6.1f}MB"
        print(line)
    for j, t in enumerate(tot):
        print(sys.argv[1 + j], {k: round(v, 1) for k, v in t.items()}, "total", round(sum(t.values()), 1))


if __name__ == "__main__":
    main()
