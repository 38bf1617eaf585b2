timeout 600 python -m pytest tests/test_executor_gpu.py -x -q 2>&1 | tail -1
timeout 600 python - <<'PY'
import sys, json, re, time
sys.path.insert(0, '.')
from paper_2304_09961_b200.executor import Executor
for suite in ("resnet50", "googlenet"):
    with Executor(suite, max_batch=90, max_requests=64) as ex:
        L = ex.desc["nets"][0]["layers"]
        base = {b: sum(ex.profile_layer(0, k, b, 5) for k in range(1, len(L) + 1)) for b in (8, 32, 90)}
        t = time.time()
        prof = ex.profile_table(batches=(1, 2, 4, 8, 16, 32, 64, 90), reps=6, tune_tiles=True)
        dt = time.time() - t
        tuned = {b: sum(ex.profile_layer(0, k, b, 5) for k in range(1, len(L) + 1)) for b in (8, 32, 90)}
        wide = sum(1 for x in prof["tile_tune"] if x[2] < 0.97 * x[3])
        print(suite, "untuned", {b: round(v, 3) for b, v in base.items()}, "tuned", {b: round(v, 3) for b, v in tuned.items()},
              "wide picks", wide, "of", len(prof["tile_tune"]), "profile+tune s %.1f" % dt, flush=True)
PY
