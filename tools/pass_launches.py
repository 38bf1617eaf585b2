"""One whole-network pass at batch b after the profile-time autotune, inside
an NVTX range "pass" (for `ncu --nvtx --nvtx-include pass/ --cache-control
none`: warm per-kernel device times of exactly that pass).

    python tools/pass_launches.py googlenet 1
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2304_09961_b200.executor import Executor  # noqa: E402

suite, b = sys.argv[1], int(sys.argv[2])
tune = os.environ.get("TUNE", "1") == "1"
with Executor(suite, max_batch=90, max_requests=4) as ex:
    L = len(ex.desc["nets"][0]["layers"])
    ex.profile_table(batches=sorted({1, 2, 4, 8, 16, 32, 64, 90, b}), reps=5, tune_tiles=tune)
    ex.profile_span(0, 1, L, b, reps=3)
    ex.sync()
    torch.cuda.nvtx.range_push("pass")
    ex.profile_span(0, 1, L, b, reps=1)
    ex.sync()
    torch.cuda.nvtx.range_pop()
