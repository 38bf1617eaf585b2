"""DRAM traffic vs algorithmic bytes per conv_tc launch over ONE population:
the config-2 workload at its measured capacity rate (profiles/r02/head/
bench_config2.json), replayed in virtual time inside a profiler range with the
executor's per-launch accounting on for every launch (every = 1). Run under
    ncu --profile-from-start off --clock-control none --metrics \
        gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv \
        --log-file OUT.csv python tools/traffic_replay.py STATS.json [requests]
then tools/traffic_summary.py OUT.csv STATS.json writes profiles/ncu_conv_summary.json
(the `traffic` bench.py reports next to its roofline)."""
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2304_09961_b200.executor import Executor  # noqa: E402

stats_out = sys.argv[1]
n_req = int(sys.argv[2]) if len(sys.argv) > 2 else 600
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
line = json.loads(open(os.path.join(root, "profiles", "r02", "head", "bench_config2.json")).read().strip().splitlines()[-1])
rate = line["config"]["offered_rate_per_gpu"]
cfg = bench.CONFIGS[2]
pk = bench.peaks()
ex = Executor(cfg["suite"], max_batch=90, max_requests=2048)
prof = ex.profile_table(batches=list(bench.BATCHES), reps=5, tune_tiles=True)
prof.pop("tile_tune", None)
job = {"profile": prof, "image_pool": 64,
       "sim": {"scheduler": cfg["scheduler"], "granularity": cfg["granularity"], "max_batch": 90},
       "workload": {"process": cfg["process"], "rate": rate, "count": n_req, "seed": 5000,
                    "relative_deadline": line["config"]["deadline_ms"]}}
ex.stats(True, every=1)
rt = ctypes.CDLL("libcudart.so.12")
rt.cudaProfilerStart()
out = ex.replay(job)
rt.cudaProfilerStop()
st = ex.stats_summary(pk["hbm_gbs"], pk["tf32_tflops"])
ex.stats(False)
json.dump({"rate": rate, "requests": n_req, "stats": st}, open(stats_out, "w"), indent=1)
print(json.dumps(st.get("conv_tc", {})))
