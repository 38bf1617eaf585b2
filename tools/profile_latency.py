"""Measures the B200 latency table h_k(b) of a suite and writes it in the
reference's profile schema (proj/include/batchsim/profile_io.hpp:3-18), the
cost model the batch-aware scheduler plans with on the GPU.

    python tools/profile_latency.py googlenet --out profiles/googlenet_b200.json
"""
from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("suite")
    ap.add_argument("--out")
    ap.add_argument("--batches", default="1,2,4,8,16,32,64,90")
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--flush-l2", action="store_true")
    ap.add_argument("--precision", default="tf32x2")
    a = ap.parse_args()
    from paper_2304_09961_b200.executor import Executor
    batches = [int(x) for x in a.batches.split(",")]
    with Executor(a.suite, max_batch=max(batches), max_requests=16) as ex:
        ex.set_precision(a.precision)
        t = time.time()
        prof = ex.profile_table(batches=batches, reps=a.reps, flush_l2=a.flush_l2)
        prof["_meta"] = {"suite": a.suite, "precision": a.precision, "flush_l2": a.flush_l2, "reps": a.reps,
                         "measured_s": round(time.time() - t, 2)}
    for comp in prof["components"]:
        tot = {b: 0.0 for b in batches}
        for L in comp["layers"]:
            for b, ms in L["runtime_ms"]:
                tot[b] += ms
        print(comp["id"], " ".join(f"b={b}:{tot[b]:.3f}ms({b / tot[b] * 1000:.0f} img/s)" for b in batches))
    if a.out:
        Path(a.out).write_text(json.dumps(prof, indent=1) + "\n")


if __name__ == "__main__":
    main()
