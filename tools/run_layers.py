"""Runs layers of one network at a fixed batch on scratch blobs (for ncu).

    python tools/run_layers.py googlenet --batch 90 --from 1 --to 22 --reps 3
"""
from __future__ import annotations

import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("suite")
    ap.add_argument("--dnn", type=int, default=0)
    ap.add_argument("--batch", type=int, default=90)
    ap.add_argument("--from", dest="lo", type=int, default=1)
    ap.add_argument("--to", dest="hi", type=int, default=0)
    ap.add_argument("--reps", type=int, default=1)
    ap.add_argument("--precision", default="tf32x2")
    a = ap.parse_args()
    from paper_2304_09961_b200.executor import Executor
    with Executor(a.suite, max_batch=max(a.batch, 1), max_requests=4) as ex:
        ex.set_precision(a.precision)
        hi = a.hi or len(ex.desc["nets"][a.dnn]["layers"])
        for k in range(a.lo, hi + 1):
            ms = ex.profile_layer(a.dnn, k, a.batch, reps=a.reps)
            print(f"layer {k} {ex.desc['nets'][a.dnn]['layers'][k - 1]['name']} b={a.batch} {ms * 1000:.1f}us")


if __name__ == "__main__":
    main()
