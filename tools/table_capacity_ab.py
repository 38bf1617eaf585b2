"""Served capacity vs the latency table's timing mode: for each mode, measure
the table, then serve a ladder of offered rates (3000 requests, two seeds)
and print on-time ratio, served req/s, drops and device / predicted time
(DEPTHS=3,4: steps in flight in the live loop).

    python tools/table_capacity_ab.py CONFIG RATE... [--modes step,pass]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2304_09961_b200.executor import Executor  # noqa: E402

args = [a for a in sys.argv[1:] if not a.startswith("--")]
modes = next((a.split("=", 1)[1] for a in sys.argv[1:] if a.startswith("--modes=")), "step,pass").split(",")
cfgn, rates = int(args[0]), [float(x) for x in args[1:]]
cfg = bench.CONFIGS[cfgn]
mb = cfg["max_batch"]
ex = Executor(cfg["suite"], max_batch=mb, max_requests=4096)
names = [n["name"] for n in ex.desc["nets"]]
sim = {"scheduler": cfg["scheduler"], "granularity": cfg["granularity"], "max_batch": mb}
if "shared_batching" in cfg:
    sim["shared_batching"] = cfg["shared_batching"]
depths = [int(x) for x in os.environ.get("DEPTHS", os.environ.get("DEPTH", "3")).split(",")]
for mode in modes:
    prof = ex.profile_table(batches=[b for b in bench.BATCHES if b < mb] + [mb], reps=10, tune_tiles=True, timing=mode)
    prof.pop("tile_tune", None)
    comp = {c["id"]: c for c in prof["components"]}
    d0 = prof["dnns"][0]
    tb = {b: sum(dict(L["runtime_ms"])[b] for cid in d0["stages"] for L in comp[cid]["layers"]) for b in (1, mb)}
    print(f"== {mode}: T1 {tb[1]:.4f} ms  T{mb} {tb[mb]:.4f} ms", flush=True)
    if os.environ.get("SAVE_TABLES"):
        json.dump(prof, open(f"{os.environ['SAVE_TABLES']}_{mode}.json", "w"))
    for depth, rate, seed in [(d, r, s) for d in depths for r in rates for s in (11, 12)]:
        if True:
            w = {"process": cfg["process"], "rate": rate, "count": 3000, "seed": seed,
                 "relative_deadline": cfg["deadline_ms"]}
            if len(names) > 1:
                w["dnn_mix"] = [[n, 1.0 / len(names)] for n in names]
            r = ex.serve({"profile": prof, "sim": sim, "image_pool": 64, "pipeline_depth": depth, "workload": w})
            print(f"  {mode} depth {depth} rate {rate:8.0f} seed {seed}: on-time {r['on_time_ratio_f']:.3f} served "
                  f"{r['served_rps']:8.0f} dropped {r['dropped']:4d} device/predicted "
                  f"{r['device_ms'] / r['predicted_step_ms_total']:.3f} steps {r['steps']}", flush=True)
