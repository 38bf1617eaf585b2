"""bin/batchsim_b200 against the reference CLI's contract
(proj/tools/batchsim_main.cpp; tests/cli_end_to_end.cmake:18-63):

* simulate: outcome CSV byte-identical to the reference's report.hpp writer
  on the same run, summary JSON identical except the wall-clock solve time;
* sweep-capacity: per-rate on-time ratio and mean completion equal to the
  reference's capacity_sweep, in the reference sweep-CSV format;
* validate-profile: sub-additivity report; oracle-check: exhaustive oracles
  agree with the DPs; exit code 2 on a bad scheduler or option; identical
  files across runs.
Fixtures: tests/golden/cli/ (tests/golden/make_cli_golden.py, from the
reference itself via oracle/_ref/ref_dump).
"""
from __future__ import annotations

import json
import struct
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
CLI = ROOT / "paper_2304_09961_b200" / "bin" / "batchsim_b200"
GOLD = ROOT / "tests" / "golden" / "cli"
SPEC = json.loads((GOLD / "cases.json").read_text())


def run(*args, ok=True):
    if not CLI.exists():
        pytest.fail("bin/batchsim_b200 is not built (python -m paper_2304_09961_b200.build)")
    r = subprocess.run([str(CLI), *map(str, args)], capture_output=True, text=True, cwd=ROOT, timeout=300)
    if ok:
        assert r.returncode == 0, r.stderr
    return r


def flags(d: dict) -> list[str]:
    out = []
    for k, v in d.items():
        out += [f"--{k}", str(v)]
    return out


def f64(h: str) -> float:
    return struct.unpack("<d", struct.pack("<Q", int(h, 16)))[0]


@pytest.mark.parametrize("case", SPEC["cases"], ids=[c[0] for c in SPEC["cases"]])
def test_simulate_matches_reference_writers(case, tmp_path):
    name, fl = case
    out = tmp_path / f"{name}.csv"
    r = run("simulate", *flags(fl), "--out", out)
    assert "on-time ratio" in r.stdout
    assert out.read_text() == (GOLD / f"{name}.csv").read_text()
    mine = json.loads((tmp_path / f"{name}.summary.json").read_text())
    ref = json.loads((GOLD / f"{name}.summary.json").read_text())
    mine.pop("mean_solve_wall_ms")
    ref.pop("mean_solve_wall_ms")
    assert mine == ref


def test_sweep_capacity_matches_reference(tmp_path):
    name, fl, scheds, rates = SPEC["sweep"]
    out = tmp_path / "sweep.csv"
    r = run("sweep-capacity", *flags(fl), "--rates", ",".join(str(x) for x in rates),
            "--schedulers", ",".join(scheds), "--out", out)
    assert "capacity[ours-time]" in r.stdout
    lines = out.read_text().splitlines()
    assert lines[0] == ("scheduler,rate,on_time_ratio_mean,on_time_ratio_std,"
                        "mean_completion_s_mean,mean_completion_s_std")
    ref = [json.loads(l) for l in (GOLD / f"{name}.sweep.jsonl").read_text().splitlines()]
    assert len(lines) - 1 == len(ref)
    for line, g in zip(lines[1:], ref):
        s, rate, ratio, rstd, comp, cstd = line.split(",")
        assert s == g["scheduler"] and float(rate) == g["rate"]
        assert ratio == "%.6f" % f64(g["ratio"]) and rstd == "0.000000"
        assert comp == "%.9f" % f64(g["mean_completion_s"]) and cstd == "0.000000000"


def test_sweep_seeds_report_spread(tmp_path):
    _, fl, _, _ = SPEC["sweep"]
    r = run("sweep-capacity", *flags(fl), "--rates", "150:450:150", "--schedulers", "ours-time", "--seeds", "3")
    rows = [l.split(",") for l in r.stdout.splitlines() if l.startswith("ours-time,")]
    assert len(rows) == 3 and all(0.0 <= float(x[2]) <= 1.0 for x in rows)


def test_validate_profile_report():
    r = run("validate-profile", "tests/golden/ref_data/googlenet.json")
    lines = r.stdout.splitlines()
    assert lines[0].startswith("component ") and "sub-additivity violations:" in lines[0]
    n = int(lines[0].rsplit(":", 1)[1])
    assert sum(1 for l in lines if l.startswith("  layer ")) == n
    assert lines[-1].startswith(f"{n} violation(s) across 1 component(s)")


@pytest.mark.parametrize("extra", [[], ["--bounded", "--max-requests", "9", "--seed", "11"]])
def test_oracle_check_passes(extra):
    r = run("oracle-check", "--instances", "150", *extra)
    assert r.stdout.strip().endswith("all oracle checks passed")
    for suite in ("completion-time DP", "tardy DP", "multi-DNN permutation search", "run-to-completion check"):
        assert f"{suite}: 150 instance(s) checked" in r.stdout


def test_exit_codes():
    assert run("simulate", "--profile", "tests/golden/ref_data/googlenet.json", "--scheduler", "bogus",
               ok=False).returncode == 2
    assert run("simulate", "--no-such-flag", "1", ok=False).returncode == 2
    assert run("frobnicate", ok=False).returncode == 2
    assert run("oracle-check", "--max-requests", "11", ok=False).returncode == 2


def test_runs_are_byte_identical(tmp_path):
    name, fl = SPEC["cases"][1]
    a, b = tmp_path / "a.csv", tmp_path / "b.csv"
    run("simulate", *flags(fl), "--out", a)
    run("simulate", *flags(fl), "--out", b)
    assert a.read_bytes() == b.read_bytes()


def test_workload_file_flags_win(tmp_path):
    wl = tmp_path / "w.json"
    wl.write_text(json.dumps({"process": "constant", "rate": 50, "requests": 40, "seed": 9}))
    r = run("simulate", "--profile", "tests/golden/ref_data/googlenet.json", "--workload", wl, "--requests", "25")
    assert "generated            25" in r.stdout
