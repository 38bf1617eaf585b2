"""Live-serving capacity (config 2) vs how the scheduler's latency table is
scaled / measured: the table measured at startup (warm), x1.05 / x1.1 / x1.2,
and a cold-L2 table; fixed deadline (default 3.559 ms) so the runs compare.

    python tools/live_scale.py [deadline_ms]
"""
import copy
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2304_09961_b200.executor import Executor  # noqa: E402

D = float(sys.argv[1]) if len(sys.argv) > 1 else 3.559
cfg = bench.CONFIGS[2]
mb = cfg["max_batch"]
ex = Executor(cfg["suite"], max_batch=mb, max_requests=4096)
batches = [b for b in bench.BATCHES if b < mb] + [mb]
warm = ex.profile_table(batches=batches, reps=10, tune_tiles=True)
warm.pop("tile_tune", None)
cold = ex.profile_table(batches=batches, reps=10, flush_l2=True)


def scaled(prof, s):
    p = copy.deepcopy(prof)
    for c in p["components"]:
        for L in c["layers"]:
            L["runtime_ms"] = [[b, t * s] for b, t in L["runtime_ms"]]
    return p


def capacity(prof, depth=2):
    sim = {"scheduler": cfg["scheduler"], "granularity": cfg["granularity"], "max_batch": mb}

    def serve(rate, i):
        w = {"process": "poisson", "rate": rate, "count": 3000, "seed": 1000 + i, "relative_deadline": D}
        r = ex.serve({"profile": prof, "sim": sim, "image_pool": 64, "pipeline_depth": depth, "workload": w})
        return r["on_time"] / r["generated"]

    cap, runs = bench.capacity_search(serve, 45000.0, 6)
    return cap, runs


for name, prof, depth in [("warm", warm, 2), ("warm x1.05", scaled(warm, 1.05), 2), ("warm x1.1", scaled(warm, 1.1), 2),
                          ("warm x1.2", scaled(warm, 1.2), 2), ("cold", cold, 2), ("warm depth 3", warm, 3),
                          ("warm depth 1", warm, 1)]:
    cap, runs = capacity(prof, depth)
    print(f"{name:14s} D={D} capacity {cap:9.1f} req/s  runs {[(round(r), round(x, 3)) for r, x in runs]}", flush=True)
