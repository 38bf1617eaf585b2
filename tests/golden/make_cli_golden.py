"""CLI/report fixtures from the REFERENCE's own writers (oracle/_ref/ref_dump
"report" and "sweep" jobs = report.hpp:35-65 on run_sim, capacity_sweep).

    python tests/golden/make_cli_golden.py

Writes tests/golden/cli/<case>.csv (outcome CSV), <case>.summary.json and
<case>.sweep.jsonl, plus cases.json (the CLI flags of every case), which
tests/test_cli.py replays through bin/batchsim_b200 and compares byte for
byte (summary: every field except the wall-clock mean_solve_wall_ms).
"""
from __future__ import annotations

import json
import subprocess
from pathlib import Path

HERE = Path(__file__).resolve().parent
ROOT = HERE.parent.parent
REF = ROOT / "oracle" / "_ref" / "ref_dump"
OUT = HERE / "cli"
D = "tests/golden/ref_data"

# (name, CLI flags, the same run as a ref_dump job)
CASES = [
    ("googlenet_time", {"profile": f"{D}/googlenet.json", "process": "poisson", "rate": 150, "requests": 400,
                        "deadline-ms": 150, "seed": 3, "scheduler": "ours-time", "granularity": "group"}),
    ("resnet50_tardy", {"profile": f"{D}/resnet50.json", "process": "pareto", "rate": 140, "requests": 400,
                        "deadline-ms": 150, "seed": 5, "scheduler": "ours-tardy", "granularity": "layer"}),
    ("five_dnns_edf", {"profile": f"{D}/five_dnns.json", "process": "poisson", "rate": 60, "requests": 300,
                       "deadline-ms": 300, "seed": 2, "scheduler": "edf", "granularity": "group"}),
    ("flow_pair_shared", {"profile": f"{D}/flow_pair.json", "process": "pareto", "rate": 40, "requests": 300,
                          "deadline-ms": 300, "seed": 4, "scheduler": "ours-time", "granularity": "group"}),
    ("googlenet_batch", {"profile": f"{D}/googlenet.json", "process": "constant", "rate": 90, "requests": 200,
                         "deadline-ms": 150, "seed": 1, "scheduler": "batch", "granularity": "group"}),
    ("collab_partial", {"profile": f"{D}/googlenet.json", "process": "pareto", "rate": 120, "requests": 300,
                        "deadline-ms": 300, "seed": 6, "scheduler": "ours-tardy", "granularity": "group",
                        "offload": "partial", "clients": 12, "client-profile": f"{D}/jetson_nano.json",
                        "trace": f"{D}/lte_uplink.csv", "trace-scale": 10}),
]
SWEEP = ("googlenet_sweep", {"profile": f"{D}/googlenet.json", "process": "poisson", "requests": 300,
                             "deadline-ms": 150, "seed": 7, "granularity": "group"},
         ["ours-time", "batch"], [100.0, 200.0, 300.0, 400.0])


def ref_job(f: dict, scheduler: str | None = None) -> dict:
    w = {"process": f["process"], "rate": f.get("rate", 100), "count": f["requests"], "seed": f["seed"]}
    if f.get("deadline-ms"):
        w["relative_deadline"] = f["deadline-ms"]
    sim = {"scheduler": scheduler or f["scheduler"], "granularity": f["granularity"]}
    for k in ("offload", "clients"):
        if k in f:
            sim[k] = f[k]
    j = {"profile": f["profile"], "workload": w, "sim": sim}
    if "trace" in f:
        j["trace"] = f["trace"]
        j["trace_scale"] = float(f["trace-scale"])
    if "client-profile" in f:
        j["client_profile"] = f["client-profile"]
    return j


def run_ref(job: dict) -> str:
    r = subprocess.run([str(REF), "-"], input=json.dumps(job), capture_output=True, text=True, cwd=ROOT)
    if r.returncode:
        raise RuntimeError(r.stderr)
    return r.stdout


def main() -> None:
    OUT.mkdir(exist_ok=True)
    for name, flags in CASES:
        text = run_ref(dict(ref_job(flags), job="report"))
        csv, summ = text.split("--\n", 1)
        (OUT / f"{name}.csv").write_text(csv)
        (OUT / f"{name}.summary.json").write_text(summ)
    name, flags, scheds, rates = SWEEP
    lines = []
    for s in scheds:
        for line in run_ref(dict(ref_job(flags, s), job="sweep", rates=rates)).splitlines():
            d = json.loads(line)
            d["scheduler"] = s
            lines.append(json.dumps(d, sort_keys=True))
    (OUT / f"{name}.sweep.jsonl").write_text("\n".join(lines) + "\n")
    (OUT / "cases.json").write_text(json.dumps({"cases": CASES, "sweep": SWEEP}, indent=1) + "\n")
    print("wrote", sorted(p.name for p in OUT.iterdir()))


if __name__ == "__main__":
    main()
