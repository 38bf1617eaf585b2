"""Measured B200 latency tables in the reference profile schema, warm (layers
inside back-to-back passes, the table bench.py plans on) and cold L2 (each
layer timed alone after an L2 flush), after the profile-time autotune.
    python tools/dump_tables.py OUTDIR googlenet resnet50_pair hetero3"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import BATCHES  # noqa: E402
from paper_2304_09961_b200.executor import Executor  # noqa: E402

out = sys.argv[1]
os.makedirs(out, exist_ok=True)
for suite in sys.argv[2:]:
    with Executor(suite, max_batch=90, max_requests=8) as ex:
        warm = ex.profile_table(batches=BATCHES, reps=10, tune_tiles=True)
        warm.pop("tile_tune", None)
        cold = ex.profile_table(batches=BATCHES, reps=10, flush_l2=True, timing="layer")
        cold.pop("tile_tune", None)
        for name, t in (("warm", warm), ("cold", cold)):
            with open(os.path.join(out, f"{suite}_table_b200_{name}.json"), "w") as f:
                json.dump(t, f, indent=1)
        print(suite, "done", flush=True)
