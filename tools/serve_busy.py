"""GPU busy fraction of the live serving loop: every layer launch timed with
events (stats every=1) during one serve run at a given rate, kernel time sum
vs the run's device time. python tools/serve_busy.py [rate] [requests]"""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2304_09961_b200.executor import Executor

rate = float(sys.argv[1]) if len(sys.argv) > 1 else 32000.0
count = int(sys.argv[2]) if len(sys.argv) > 2 else 3000
depth = int(sys.argv[3]) if len(sys.argv) > 3 else 2
ex = Executor("googlenet", max_batch=90, max_requests=4096)
prof = ex.profile_table(batches=[1, 2, 4, 8, 16, 32, 64, 90], reps=10)
base = {"profile": prof, "sim": {"scheduler": "ours-tardy", "granularity": "layer", "max_batch": 90},
        "image_pool": 64, "pipeline_depth": depth}
job = dict(base, workload={"process": "poisson", "rate": rate, "count": count, "seed": 7, "relative_deadline": 5.0},
           h2d=False)
ex.serve(job)  # warm
ex.stats(True, every=1)
r = ex.serve(job)
ex.sync()
s = ex.stats_summary(6550.0, 696.0)
ex.stats(False)
busy = sum(v["ms"] for v in s.values() if isinstance(v, dict) and "ms" in v)
launches = sum(v["launches"] for v in s.values() if isinstance(v, dict) and "launches" in v)
print(json.dumps({k: r[k] for k in r if not isinstance(r[k], (list, dict))}))
print(f"depth {depth} rate {rate}: on-time {r['on_time_ratio_f']:.4f} served {r['served_rps']:.0f}, device_ms {r['device_ms']:.1f}, timed kernels {launches}, kernel ms {busy:.1f}, "
      f"busy {busy / r['device_ms']:.3f}")
