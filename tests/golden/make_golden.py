"""Regenerates the schedule-parity fixtures from the REFERENCE (oracle/_ref/ref_dump,
built by oracle/Makefile from /root/reference's headers).

    python tests/golden/make_golden.py

Writes
  tests/golden/sched_sim.json        sim jobs + sha256 of the reference's full
                                      plan/step/outcome trace + its summary line
  tests/golden/sched_calls.jsonl.gz  random instances (reference.hpp:286-339
                                      generators) + the reference's result for
                                      every scheduler call on them

Profiles / client profile / LTE trace are the reference's data files, copied
verbatim as fixtures under tests/golden/ref_data/ (data, not code).
"""
from __future__ import annotations

import gzip
import hashlib
import json
import subprocess
import sys
import tempfile
from pathlib import Path

HERE = Path(__file__).resolve().parent
ROOT = HERE.parent.parent
REF = ROOT / "oracle" / "_ref" / "ref_dump"
DATA = "tests/golden/ref_data"  # relative to the repo root (tests chdir there)


def canon_lines(text: str) -> list[str]:
    out = []
    for line in text.splitlines():
        d = json.loads(line)
        d.pop("wall_ms", None)
        out.append(json.dumps(d, sort_keys=True, separators=(",", ":")))
    return out


def digest(lines: list[str]) -> str:
    h = hashlib.sha256()
    for l in lines:
        h.update(l.encode())
        h.update(b"\n")
    return h.hexdigest()


def run_ref(job: dict) -> str:
    with tempfile.NamedTemporaryFile("w", suffix=".json", delete=False) as f:
        json.dump(job, f)
        path = f.name
    r = subprocess.run([str(REF), path], capture_output=True, text=True, cwd=ROOT)
    if r.returncode != 0:
        raise RuntimeError(r.stderr)
    return r.stdout


MIX5 = [["vgg16", .2], ["resnet50", .2], ["fcn", .2], ["googlenet", .2], ["ssd", .2]]
MIXF = [["sdcnet", .5], ["rta", .5]]


def sim_jobs() -> list[tuple[str, dict]]:
    jobs = []
    for prof, mix, dl in [("googlenet", None, 150), ("resnet50", None, 150), ("five_dnns", MIX5, 150),
                          ("flow_pair", MIXF, 300)]:
        for sched in ["ours-time", "ours-tardy", "edf", "batch", "no-batch"]:
            for gran in ["group", "layer", "request"]:
                for proc, rate in [("poisson", 150), ("pareto", 90), ("constant", 60)]:
                    if gran == "request" and proc != "poisson":
                        continue
                    w = {"process": proc, "rate": rate, "count": 200, "seed": 3, "relative_deadline": dl}
                    if mix:
                        w["dnn_mix"] = mix
                    jobs.append((f"{prof}-{sched}-{gran}-{proc}",
                                 {"job": "sim", "profile": f"{DATA}/{prof}.json", "workload": w,
                                  "sim": {"scheduler": sched, "granularity": gran}}))
    for off in ["binary", "partial"]:
        for sched in ["ours-time", "ours-tardy"]:
            jobs.append((f"collab-{off}-{sched}",
                         {"job": "sim", "profile": f"{DATA}/five_dnns.json",
                          "workload": {"process": "pareto", "rate": 120, "count": 300, "seed": 5,
                                       "relative_deadline": 150, "dnn_mix": [["vgg16", .5], ["fcn", .5]]},
                          "sim": {"scheduler": sched, "granularity": "group", "offload": off, "clients": 12},
                          "trace": f"{DATA}/lte_uplink.csv", "trace_scale": 10,
                          "client_profile": f"{DATA}/jetson_nano.json"}))
    jobs.append(("googlenet-window-latency-overhead",
                 {"job": "sim", "profile": f"{DATA}/googlenet.json",
                  "workload": {"process": "poisson", "rate": 400, "count": 600, "seed": 9},
                  "sim": {"scheduler": "ours-time", "granularity": "layer", "window_cap": 50,
                          "scheduler_latency": 0.7, "step_overhead": 0.3}}))
    jobs.append(("flow-pair-no-shared-batching",
                 {"job": "sim", "profile": f"{DATA}/flow_pair.json",
                  "workload": {"process": "poisson", "rate": 80, "count": 300, "seed": 2, "dnn_mix": MIXF},
                  "sim": {"scheduler": "ours-time", "granularity": "group", "shared_batching": False}}))
    jobs.append(("googlenet-constant-net-10mbps",
                 {"job": "sim", "profile": f"{DATA}/googlenet.json",
                  "workload": {"process": "constant", "rate": 30, "count": 50, "seed": 1},
                  "sim": {"scheduler": "ours-time", "granularity": "request"},
                  "trace_points": [[0.0, 10000.0]]}))
    # closed instances (explicit arrivals), reference test_simulator.cpp:13-19
    jobs.append(("googlenet-closed-10",
                 {"job": "sim", "profile": f"{DATA}/googlenet.json",
                  "workload": {"explicit_arrivals": [[0.0, 0, 200000]] * 10},
                  "sim": {"scheduler": "ours-time", "granularity": "request"}}))
    return jobs


FNS_SINGLE = ([{"fn": "dp", "granularity": g, "groups": G} for g in ("request", "layer", "group") for G in (2, 3)]
              + [{"fn": "tardy", "granularity": g, "groups": 2, "now": 5.0} for g in ("request", "layer", "group")]
              + [{"fn": "tardy", "granularity": "request", "now": 3.0, "start_offset": 7.5},
                 {"fn": "edf", "now": 2.0}, {"fn": "batch"}, {"fn": "no_batch"},
                 {"fn": "dp", "granularity": "request", "bound": 2},
                 {"fn": "segment", "layers": [3, 1, 2, 1]}, {"fn": "groups", "groups": 1}, {"fn": "lookup"},
                 {"fn": "dp", "granularity": "group", "groups": 3, "extra_active": 4}])
FNS_MULTI = ([{"fn": "multi", "granularity": g, "groups": 2} for g in ("request", "layer", "group")]
             + [{"fn": "multi_shared", "granularity": "request"},
                {"fn": "multi", "granularity": "request", "guard": 1, "heuristic": False}])


def random_jobs() -> list[dict]:
    jobs = []
    for style in ("arbitrary", "subadditive", "strong"):
        for dl in (False, True):
            jobs.append({"job": "random", "seed": 11 + len(jobs), "trials": 40, "max_requests": 9,
                         "max_layers": 6, "style": style, "deadlines": dl, "fns": FNS_SINGLE})
            jobs.append({"job": "random", "seed": 101 + len(jobs), "trials": 30, "max_requests": 3,
                         "max_layers": 4, "style": style, "deadlines": dl, "dnns": 3, "fns": FNS_MULTI})
    return jobs


def shared_pair_calls() -> dict:
    """The hand-built shared-prefix pair of test_multidnn.cpp:68-94, with
    interleaved arrivals (riders must appear)."""
    comp = lambda cid, grid, n: {"id": cid, "layers": [{"output_bits": 500000, "runtime_ms": grid}] * n}
    prof = {"max_batch": 90,
            "components": [comp("flow", [[1, 10.0], [2, 11.0], [3, 12.0], [4, 13.0]], 2),
                           comp("head_a", [[1, 2.0], [2, 2.2], [3, 2.4], [4, 2.6]], 1),
                           comp("head_b", [[1, 2.0], [2, 2.2], [3, 2.4], [4, 2.6]], 1)],
            "dnns": [{"id": "task_a", "stages": ["flow", "head_a"]}, {"id": "task_b", "stages": ["flow", "head_b"]}]}
    calls = []
    reqsets = [[[1, 0, 0.0, None, 1], [2, 1, 1.0, None, 1]],
               [[1, 0, 0.0, None, 1], [2, 1, 1.0, None, 1], [3, 0, 2.0, None, 1], [4, 1, 3.0, None, 1]],
               [[1, 1, 0.0, None, 2], [2, 0, 1.0, None, 1], [3, 1, 2.0, None, 1]]]
    for reqs in reqsets:
        for fn in ("multi", "multi_shared"):
            for g in ("request", "layer"):
                calls.append({"fn": fn, "granularity": g, "requests": reqs})
    return {"job": "calls", "profile": prof, "calls": calls}


def main() -> None:
    if not REF.exists():
        sys.exit(f"{REF} missing: run `make -C oracle` (needs /root/reference)")
    sims = []
    for name, job in sim_jobs():
        lines = canon_lines(run_ref(job))
        sims.append({"name": name, "job": job, "lines": len(lines), "sha256": digest(lines),
                     "summary": json.loads(lines[-1])})
    (HERE / "sched_sim.json").write_text(json.dumps(sims, indent=1) + "\n")
    n_calls = 0
    with gzip.open(HERE / "sched_calls.jsonl.gz", "wt") as f:
        for job in random_jobs():
            for line in run_ref(job).splitlines():
                f.write(line + "\n")
                n_calls += len(json.loads(line)["calls"])
        sp = shared_pair_calls()
        out = [json.loads(l) for l in run_ref(sp).splitlines()]
        f.write(json.dumps({"trial": -1, "profile": sp["profile"], "requests": None, "calls": out}) + "\n")
        n_calls += len(out)
    print(f"{len(sims)} sim traces, {n_calls} scheduler calls")


if __name__ == "__main__":
    main()
