"""Live capacity with the scheduler's latency table timed per layer alone
(synchronised) vs inside back-to-back passes, per config, at the committed
deadline; plus the table's predicted vs executed step time.

    python tools/table_timing_ab.py 2 4 3 1
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2304_09961_b200.executor import Executor  # noqa: E402

for cfgn in [int(x) for x in sys.argv[1:]] or [2, 4]:
    cfg = bench.CONFIGS[cfgn]
    mb = cfg["max_batch"]
    ex = Executor(cfg["suite"], max_batch=mb, max_requests=4096)
    batches = [b for b in bench.BATCHES if b < mb] + [mb]
    tabs = {}
    tabs["layer"] = ex.profile_table(batches=batches, reps=10, tune_tiles=True, timing="layer")
    tabs["layer"].pop("tile_tune", None)
    tabs["pass"] = ex.profile_table(batches=batches, reps=10, timing="pass")
    D = round(cfg.get("deadline_t1_factor", 6.25) * bench.committed_t1(cfgn), 3)
    names = [n["name"] for n in ex.desc["nets"]]
    for name, prof in tabs.items():
        comp = {c["id"]: c for c in prof["components"]}
        t = {b: max(sum(dict(L["runtime_ms"])[b] for cid in d["stages"] for L in comp[cid]["layers"])
                    for d in prof["dnns"]) for b in (1, mb)}

        def serve(rate, i, detail=None):
            w = {"process": cfg["process"], "rate": rate, "count": 3000, "seed": 1000 + i, "relative_deadline": D}
            if len(names) > 1:
                w["dnn_mix"] = [[n, 1.0 / len(names)] for n in names]
            job = dict(bench.collab_inputs(cfg), profile=prof, sim=bench.sim_config(cfg, mb), image_pool=64,
                       pipeline_depth=2, workload=w)
            r = ex.serve(job)
            if detail is not None:
                detail.append(r)
            return r["on_time"] / r["generated"]

        cap, runs = bench.capacity_search(serve, mb / t[mb] * 1000.0, 6)
        det = []
        serve(cap, 99, det)
        r = det[0]
        print(f"config {cfgn} table={name:5s} T1 {t[1]:.3f} T{mb} {t[mb]:.3f} ms D={D}: capacity {cap:9.1f} "
              f"runs {[(round(x), round(y, 3)) for x, y in runs]} | at cap: device {r['device_ms']:.1f} ms "
              f"predicted steps {r['predicted_step_ms_total']:.1f} ms", flush=True)
    ex.close()
