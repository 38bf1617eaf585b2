"""Kernel mix of the timed workload for an ncu launch list: config 2 at its
measured capacity rate (bench_config2.json), replayed in virtual time (every
step executed; under ncu the live loop cannot keep its deadlines), inside a
profiler range.
    ncu --profile-from-start off --metrics gpu__time_duration.sum --csv ... python tools/launch_list_replay.py [requests]"""
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2304_09961_b200.executor import Executor  # noqa: E402

n_req = int(sys.argv[1]) if len(sys.argv) > 1 else 600
line = json.load(open(os.path.join(os.path.dirname(__file__), "..", "profiles", "r02", "bench_config2.json")))
rate = line["config"]["offered_rate_per_gpu"]
cfg = bench.CONFIGS[2]
ex = Executor(cfg["suite"], max_batch=90, max_requests=2048)
prof = ex.profile_table(batches=list(bench.BATCHES), reps=5, tune_tiles=True)
prof.pop("tile_tune", None)
job = {"profile": prof, "image_pool": 64,
       "sim": {"scheduler": cfg["scheduler"], "granularity": cfg["granularity"], "max_batch": 90},
       "workload": {"process": cfg["process"], "rate": rate, "count": n_req, "seed": 5000,
                    "relative_deadline": line["config"]["deadline_ms"]}}
rt = ctypes.CDLL("libcudart.so.12")
rt.cudaProfilerStart()
out = ex.replay(job)
rt.cudaProfilerStop()
print(json.dumps(out[-1] if isinstance(out, list) else out)[:400])
