"""Whole-network pass times at several batches: synchronised (host launch
latency included), back-to-back eager launches, and one CUDA graph replayed.

    python tools/span_bench.py small_cnn:1,10 googlenet:1,8,32,90
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2304_09961_b200.executor import Executor  # noqa: E402

for arg in sys.argv[1:] or ["small_cnn:1,10", "googlenet:1,8,32,90"]:
    suite, bs = arg.split(":")
    prec = os.environ.get("BS_PREC", "tf32x2")
    with Executor(suite, max_batch=90, max_requests=4) as ex:
        ex.set_precision(prec)
        L = len(ex.desc["nets"][0]["layers"])
        for b in [int(x) for x in bs.split(",")]:
            s, e, g = ex.profile_span(0, 1, L, b, reps=30)
            print(f"{suite} b={b} layers 1-{L}: sync {s * 1000:.1f} us  back-to-back {e * 1000:.1f} us  "
                  f"graph {g * 1000:.1f} us", flush=True)
