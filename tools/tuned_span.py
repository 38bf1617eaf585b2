"""Whole-network pass times after the profile-time autotune (K split, tile
width, grouping), next to the launcher's untuned rules: per batch the sum
of the measured per-layer latencies (the scheduler's table) and one pass
as a CUDA graph / back-to-back eager launches.

    python tools/tuned_span.py googlenet:1,8,32,90 resnet50:1,8
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2304_09961_b200.executor import Executor  # noqa: E402

BATCHES = (1, 2, 4, 8, 12, 16, 24, 32, 48, 64, 90)
for arg in sys.argv[1:] or ["googlenet:1,8,32,90"]:
    suite, bs = arg.split(":")
    want = [int(x) for x in bs.split(",")]
    with Executor(suite, max_batch=90, max_requests=4) as ex:
        L = len(ex.desc["nets"][0]["layers"])
        res = {}
        for tuned in (False, True):
            batches = sorted(set(BATCHES) | set(want))
            prof = ex.profile_table(batches=batches, reps=10, tune_tiles=tuned)
            tl = prof.pop("tile_tune", None)
            comp = {c["id"]: c for c in prof["components"]}
            d = prof["dnns"][0]
            for b in want:
                s = sum(dict(Lr["runtime_ms"])[b] for cid in d["stages"] for Lr in comp[cid]["layers"])
                sync, eager, graph = ex.profile_span(0, 1, L, b, reps=30)
                res.setdefault(b, {})["tuned" if tuned else "rules"] = (s * 1000, eager * 1000, graph * 1000)
            if tuned and tl is not None and os.environ.get("TUNE_LOG"):
                with open(os.environ["TUNE_LOG"] + f".{suite}.json", "w") as f:
                    json.dump(tl, f)
        for b in want:
            r = res[b]
            print(f"{suite} b={b}: layer-sum rules {r['rules'][0]:.1f} tuned {r['tuned'][0]:.1f} us | "
                  f"pass eager {r['rules'][1]:.1f} -> {r['tuned'][1]:.1f} us | graph {r['rules'][2]:.1f} -> "
                  f"{r['tuned'][2]:.1f} us", flush=True)
