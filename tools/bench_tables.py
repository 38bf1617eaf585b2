"""The B200 latency tables bench.py plans on, measured the way bench.py does at
startup (profile-time autotune, then bench.table_timing(cfg): each layer as a
one-layer serving step for layer granularity, inside whole passes otherwise), one per bench config, in the reference profile
schema -- committed as profiles/r02/*_table_b200.json for the reference arm.
    python tools/bench_tables.py OUTDIR [config ...]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2304_09961_b200.executor import Executor  # noqa: E402

out = sys.argv[1]
os.makedirs(out, exist_ok=True)
for c in [int(x) for x in sys.argv[2:]] or sorted(bench.CONFIGS):
    cfg = bench.CONFIGS[c]
    mb = cfg["max_batch"]
    with Executor(cfg["suite"], max_batch=mb, max_requests=8) as ex:
        timing = bench.table_timing(cfg)
        prof = ex.profile_table(batches=[b for b in bench.BATCHES if b < mb] + [mb], reps=10, tune_tiles=True,
                                timing=timing)
        prof.pop("tile_tune", None)
        how = ("each layer a one-layer serving step (pointer-table kernel + layer) in back-to-back step "
               "passes, device-stamped" if timing == "step" else
               "per-layer events inside back-to-back passes scaled to the whole-pass time")
        prof["_meta"] = {"measured": "tools/bench_tables.py on one B200 (bench.py's startup table: autotuned "
                                     f"launches, {how}, median of 10)", "precision": "tf32x2", "suite": cfg["suite"]}
        path = os.path.join(out, f"{cfg['suite']}_table_b200.json")
        with open(path, "w") as f:
            json.dump(prof, f, indent=1)
        print(c, path, flush=True)
