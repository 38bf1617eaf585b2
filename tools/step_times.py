"""Per-step device time vs the latency table's prediction in the live loop
(BS_LIVE_STEP_TIMES=1: a timing event after every step).

    python tools/step_times.py CONFIG RATE [out.json]

Prints actual/predicted by step batch size and by the number of steps in
flight when the step was launched (0 = the GPU may have idled before it)."""
import json
import os
import sys

os.environ.setdefault("BS_LIVE_STEP_TIMES", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2304_09961_b200.executor import Executor  # noqa: E402

cfgn, rate = int(sys.argv[1]), float(sys.argv[2])
cfg = bench.CONFIGS[cfgn]
mb = cfg["max_batch"]
ex = Executor(cfg["suite"], max_batch=mb, max_requests=4096)
prof = ex.profile_table(batches=[b for b in bench.BATCHES if b < mb] + [mb], reps=10, tune_tiles=True)
prof.pop("tile_tune", None)
names = [n["name"] for n in ex.desc["nets"]]
sim = {"scheduler": cfg["scheduler"], "granularity": cfg["granularity"], "max_batch": mb}
if "shared_batching" in cfg:
    sim["shared_batching"] = cfg["shared_batching"]
w = {"process": cfg["process"], "rate": rate, "count": 3000, "seed": 11,
     "relative_deadline": float(os.environ.get("DEADLINE_MS", cfg["deadline_ms"]))}
if len(names) > 1:
    w["dnn_mix"] = [[n, 1.0 / len(names)] for n in names]
job = {"profile": prof, "sim": sim, "image_pool": 64, "pipeline_depth": int(os.environ.get("DEPTH", "3")), "workload": w}
r = ex.serve(job)
rows = r.pop("step_times", [])
print(json.dumps({k: r[k] for k in ("offered_rps", "served_rps", "on_time_ratio_f", "device_ms",
                                     "predicted_step_ms_total", "steps", "dropped")}))
if len(sys.argv) > 3:
    json.dump({"summary": {k: v for k, v in r.items() if not isinstance(v, (list, dict))}, "rows": rows},
              open(sys.argv[3], "w"))
# rows: from, to, batch, predicted, in flight at launch, new members, finishing, riders, device ms
if not rows:
    sys.exit(0)
tot_p = sum(x[3] for x in rows)
tot_a = sum(x[8] for x in rows)
print(f"steps {len(rows)} predicted {tot_p:.2f} ms device {tot_a:.2f} ms ratio {tot_a / tot_p:.3f}")
keys = [("in flight at launch", lambda x: int(x[4])), ("layers", lambda x: int(x[1] - x[0] + 1)),
        ("has new members", lambda x: int(x[5] > 0)), ("has finishing", lambda x: int(x[6] > 0)),
        ("riders in step", lambda x: int(x[7])),
        ("layer", lambda x: int(x[0]))]
if os.environ.get("BY_BATCH"):
    keys.append(("batch", lambda x: int(x[2])))
for key, f in keys:
    agg = {}
    for x in rows:
        a = agg.setdefault(f(x), [0, 0.0, 0.0])
        a[0] += 1
        a[1] += x[3]
        a[2] += x[8]
    print(key)
    for k in sorted(agg):
        n, p, a = agg[k]
        print(f"  {k:4d}: n {n:5d} predicted {p:8.2f} device {a:8.2f} ratio {a / max(p, 1e-9):.3f} excess/step {(a - p) / n * 1000:7.1f} us")
