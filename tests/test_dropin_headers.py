"""Drop-in include shims (include/batchsim/*.hpp): reference-style user code
written against <batchsim/batchsim.hpp> builds unchanged with -I<repo>/include
and links libbs_host.so (CPU only). When the reference is mounted the same
source is also built against the reference headers and both runs print the
same results."""
import subprocess
from pathlib import Path

import pytest

from paper_2304_09961_b200.build import JSON_INC

ROOT = Path(__file__).resolve().parent.parent
SRC = ROOT / "tests" / "dropin" / "user_sim.cpp"
LIB = ROOT / "paper_2304_09961_b200" / "lib"
PROFILE = ROOT / "tests" / "golden" / "ref_data" / "googlenet.json"
REF_INC = Path("/root/reference/proj/include")


def build_and_run(tmp_path, name, incs, libs):
    exe = tmp_path / name
    cmd = ["g++", "-std=c++20", "-O1", *[f"-I{i}" for i in incs], f"-I{JSON_INC}", str(SRC), "-o", str(exe), *libs]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    return subprocess.run([str(exe), str(PROFILE)], check=True, capture_output=True, text=True).stdout


def test_shims_cover_every_reference_header():
    shims = {p.name for p in (ROOT / "include" / "batchsim").glob("*.hpp")}
    assert {"batchsim.hpp", "simulator.hpp", "dp_time.hpp", "deadline.hpp", "multi_dnn.hpp", "cost_model.hpp",
            "profile_io.hpp", "schedule.hpp", "workload.hpp", "network.hpp", "offload.hpp", "rng.hpp",
            "model.hpp", "report.hpp", "reference.hpp"} <= shims
    if REF_INC.exists():
        assert {p.name for p in (REF_INC / "batchsim").glob("*.hpp")} <= shims


def test_reference_style_code_builds_against_the_shims(tmp_path):
    out = build_and_run(tmp_path, "ours", [ROOT / "include"],
                        [f"-L{LIB}", "-lbs_host", f"-Wl,-rpath,{LIB}"])
    assert out.splitlines()[-1] == "ok", out
    if REF_INC.exists():
        assert build_and_run(tmp_path, "ref", [REF_INC], []) == out
