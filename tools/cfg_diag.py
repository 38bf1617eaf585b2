"""Diagnoses the multi-DNN serving configs (3: ResNet-50 pair with shared
riders, Pareto; 4: hetero3, Poisson): serve at a ladder of offered rates and
print the loop's host/device accounting per run.

    python tools/cfg_diag.py 3 1000 2000 4000 8000
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2304_09961_b200.executor import Executor  # noqa: E402

cfgn = int(sys.argv[1])
DEPTH = int(os.environ.get("DEPTH", "2"))
D_OVERRIDE = float(os.environ["DEADLINE_MS"]) if os.environ.get("DEADLINE_MS") else None
rates = [float(x) for x in sys.argv[2:]] or [1000, 2000, 4000]
cfg = bench.CONFIGS[cfgn]
mb = cfg["max_batch"]
ex = Executor(cfg["suite"], max_batch=mb, max_requests=4096)
prof = ex.profile_table(batches=[b for b in bench.BATCHES if b < mb] + [mb], reps=10, tune_tiles=True)
prof.pop("tile_tune", None)
names = [n["name"] for n in ex.desc["nets"]]
comp = {c["id"]: c for c in prof["components"]}


def dnn_ms(d, b):
    return sum(dict(L["runtime_ms"])[b] for cid in d["stages"] for L in comp[cid]["layers"])


for d in prof["dnns"]:
    print(d["id"], "T1 %.3f ms  T%d %.3f ms" % (dnn_ms(d, 1), mb, dnn_ms(d, mb)))
t1 = max(dnn_ms(d, 1) for d in prof["dnns"])
deadline = D_OVERRIDE or round(6.25 * t1, 3)
sim = {"scheduler": cfg["scheduler"], "granularity": cfg["granularity"], "max_batch": mb}
if "shared_batching" in cfg:
    sim["shared_batching"] = cfg["shared_batching"]
for proc in ([cfg["process"], "poisson"] if cfg["process"] != "poisson" else ["poisson"]):
    for rate in rates:
        w = {"process": proc, "rate": rate, "count": 3000, "seed": 11, "relative_deadline": deadline}
        if len(names) > 1:
            w["dnn_mix"] = [[n, 1.0 / len(names)] for n in names]
        job = {"profile": prof, "sim": sim, "image_pool": 64, "pipeline_depth": DEPTH, "workload": w}
        stats = os.environ.get("STATS", "1") == "1"  # per-launch events break PDL chains
        ex.stats(stats, every=1)
        r = ex.serve(job)
        s = ex.stats_summary(6550.0, 696.0) if stats else {}
        ex.stats(False)
        busy = sum(v["ms"] for v in s.values() if isinstance(v, dict) and "ms" in v)
        keep = {k: (round(v, 3) if isinstance(v, float) else v) for k, v in r.items() if not isinstance(v, (list, dict)) or k == "step_members_hist"}
        keep["kernel_over_predicted"] = round(busy / max(r["predicted_step_ms_total"], 1e-9), 3)
        keep["kernel_ms"] = round(busy, 2)
        keep["busy_frac"] = round(busy / max(r["device_ms"], 1e-9), 3)
        print(proc, "deadline", deadline, json.dumps(keep), flush=True)
