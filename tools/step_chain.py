"""Cost of the serving loop's per-step extras on a whole-network pass run as
one-layer steps (executor profile_span with BS_SPAN_STEP): 0 plain PDL
chain, 1 + a table-write kernel per layer, 4 + an event record per layer,
5 both, 8 + the table by H2D on a side stream and a cross-stream wait, 12
that + an event.

    python tools/step_chain.py googlenet 1 10 40 90
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2304_09961_b200.executor import Executor  # noqa: E402

suite = sys.argv[1]
bs = [int(x) for x in sys.argv[2:]] or [1, 10, 40, 90]
with Executor(suite, max_batch=90, max_requests=4) as ex:
    L = len(ex.desc["nets"][0]["layers"])
    ex.profile_table(batches=sorted(set([1, 2, 4, 8] + bs)), reps=5, tune_tiles=True)
    for b in bs:
        row = []
        for bits in (0, 1, 4, 5, 8, 12, 0):
            os.environ["BS_SPAN_STEP"] = str(bits)
            _, e, _ = ex.profile_span(0, 1, L, b, reps=30)
            row.append(f"{bits}:{e * 1e3:8.1f}")
        print(f"{suite} b={b:3d} layers {L}  " + "  ".join(row) + "  us/pass", flush=True)
