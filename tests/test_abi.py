"""The C-ABI libraries load on a host without a GPU and export every entry
point declared in include/*.h (no compute calls here)."""
import ctypes
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent


def declared(header: str) -> list[str]:
    text = (ROOT / "include" / header).read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+[\s\*]+(bs_\w+)\s*\(", text, flags=re.M)))


@pytest.mark.parametrize("header,lib", [("bs_exec.h", "libbs_exec.so"), ("bs_host.h", "libbs_host.so"),
                                        ("bs_nets.h", "libbs_nets.so")])
def test_library_exports_header(header, lib):
    names = declared(header)
    assert len(names) >= 3
    so = ctypes.CDLL(str(ROOT / "paper_2304_09961_b200" / "lib" / lib))
    missing = [n for n in names if not hasattr(so, n)]
    assert not missing, missing


def test_describe_suite_without_gpu():
    from paper_2304_09961_b200.executor import describe_suite
    d = describe_suite("googlenet")
    net = d["nets"][0]
    assert len(net["layers"]) == 22  # reference profile: googlenet.json has 22 layers
    params = sum(o["weight_floats"] for o in net["ops"])
    assert 6.5e6 < params < 6.7e6
    gflops = sum(o["flops"] for o in net["ops"]) / 1e9
    assert abs(gflops - 3.0) < 0.05


@pytest.mark.parametrize("suite,layers", [("small_cnn", [5]), ("resnet50", [50]), ("mobilenet_v2", [53]),
                                          ("resnet50_pair", [50, 51]), ("hetero3", [22, 50, 53])])
def test_suite_layer_counts(suite, layers):
    from paper_2304_09961_b200.executor import describe_suite
    d = describe_suite(suite)
    assert [len(n["layers"]) for n in d["nets"]] == layers


def test_shared_backbone_planned_identically():
    from paper_2304_09961_b200.executor import describe_suite
    d = describe_suite("resnet50_pair")
    a, b = d["nets"]
    for L in range(49):  # the shared component: same ops, offsets, weights
        oa = [a["ops"][i] for i in a["layers"][L]["ops"]]
        ob = [b["ops"][i] for i in b["layers"][L]["ops"]]
        for x, y in zip(oa, ob):
            assert x["w_off"] == y["w_off"]
            assert a["tensors"][x["out"][0]]["off"] == b["tensors"][y["out"][0]]["off"]


def test_missing_library_is_an_error(monkeypatch, tmp_path):
    from paper_2304_09961_b200 import _native
    monkeypatch.setattr(_native, "LIB_DIR", tmp_path)
    monkeypatch.setattr(_native, "_exec", None)
    with pytest.raises(_native.BsError):
        _native.exec_lib()
