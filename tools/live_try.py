import json, sys, time
sys.path.insert(0, '/root/repo')
from paper_2304_09961_b200.executor import Executor
prof = json.load(open('gpurun_out/googlenet_b200.json'))
t1 = sum(L["runtime_ms"][0][1] for L in prof["components"][0]["layers"])
print("T1 ms", t1)
with Executor("googlenet", max_batch=90, max_requests=2048) as ex:
    for rate in [500, 2000, 5000, 10000, 20000]:
        job = {"profile": prof, "workload": {"process": "poisson", "rate": rate, "count": 3000, "seed": 3, "relative_deadline": 6.25 * t1},
               "sim": {"scheduler": "ours-tardy", "granularity": "layer"}, "image_pool": 32}
        t = time.time(); r = ex.serve(job)
        print(rate, {k: r[k] for k in ("completed", "dropped", "on_time_ratio_f", "served_rps", "goodput_rps", "mean_completion_ms", "p95_completion_ms", "steps", "plans", "sched_ms_total", "sched_ms_max", "launches", "wall_ms")}, round(time.time()-t,1))
