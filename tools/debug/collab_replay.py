"""Config-5 replay: every server-finished request against the oracle, with
its outcome record (location, offload groups)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
os.chdir(ROOT)
import numpy as np
from oracle.forward import NetOracle, rel_err
from paper_2304_09961_b200.executor import Executor
from test_executor_gpu import synth_profile, image_for

pool = int(sys.argv[1]) if len(sys.argv) > 1 else 0
with Executor("collab", max_batch=90, max_requests=64) as ex:
    w = ex.weights()
    orcs = [NetOracle(ex.desc, k, w) for k in range(2)]
    names = [n["name"] for n in ex.desc["nets"]]
    job = {"profile": synth_profile(ex, 1.0, 0.02),
           "workload": {"process": "pareto", "rate": 60, "count": 24, "seed": 11,
                        "dnn_mix": [[n, 0.5] for n in names]},
           "sim": {"scheduler": "ours-time", "granularity": "group", "max_batch": 90,
                   "offload": "partial", "clients": 4},
           "client_profile": "tests/golden/ref_data/jetson_nano.json",
           "trace": "tests/golden/ref_data/lte_uplink.csv", "trace_scale": 10.0,
           "image_seed": 9, "dump_ids": list(range(1, 25)), "image_pool": pool}
    out = ex.replay(job)
    outcomes = next(r for r in out if r["ev"] == "outcomes")["outcomes"]
    res = next(r for r in out if r["ev"] == "results")
    for o in outcomes:
        rid, dnn, loc, groups = o[0], o[1], o[7], o[8]
        if loc == 1:
            print(rid, names[dnn], "client_full"); continue
        idx = (rid - 1) % pool if pool else rid - 1
        ref = orcs[dnn].probs(orcs[dnn].forward(image_for(ex, dnn, idx, seed=9)))
        got = np.array(res["probs"][str(rid)], np.float32)[:ref.size]
        print(rid, names[dnn], "loc", loc, "groups", groups, "err %.2e" % rel_err(got, ref), flush=True)
