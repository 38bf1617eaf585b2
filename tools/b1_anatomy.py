"""Small-batch pass anatomy: pass times (sync / eager / graph) after the
profile-time autotune, and (mode "ncu") a few eager passes to run under
`ncu --cache-control none` for warm per-kernel durations.

    python tools/b1_anatomy.py googlenet 1 [ncu]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2304_09961_b200.executor import Executor  # noqa: E402

suite, b = sys.argv[1], int(sys.argv[2])
mode = sys.argv[3] if len(sys.argv) > 3 else "time"
with Executor(suite, max_batch=90, max_requests=4) as ex:
    L = len(ex.desc["nets"][0]["layers"])
    ex.profile_table(batches=sorted({1, 2, 4, 8, b}), reps=5, tune_tiles=True)
    if mode == "ncu":
        # run under `ncu --profile-from-start off`: only the passes below
        import ctypes
        rt = ctypes.CDLL("libcudart.so.12")
        rt.cudaProfilerStart()
        ex.profile_span(0, 1, L, b, reps=1)
        rt.cudaProfilerStop()
    else:
        s, e, g = ex.profile_span(0, 1, L, b, reps=50)
        print(f"{suite} b={b} pdl={os.environ.get('BS_PDL', '1')}: sync {s * 1e3:.1f} eager {e * 1e3:.1f} "
              f"graph {g * 1e3:.1f} us  launches/pass {ex.launches_per_pass if hasattr(ex, 'launches_per_pass') else '?'}",
              flush=True)
