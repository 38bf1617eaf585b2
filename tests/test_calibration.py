"""Synthetic-weight acceptance and the layer oracle pinned to
PyTorch — CPU only.

* oracle/layers.py + oracle/forward.py (numpy, per image) agree with
  torch.nn.functional (conv2d, max_pool2d(ceil_mode), mean, softmax;
  oracle/torch_forward.py) on every op output of every network.
* The calibrated weights (csrc/exec/calib.cpp) give input-dependent outputs:
  >= 50 distinct top-1 classes over 256 random inputs for GoogLeNet,
  ResNet-50 and MobileNetV2 (all 10 for SmallCNN), per-layer RMS in
  [0.1, 10], and logits whose spread across inputs dominates their
  calibration-batch mean (so the 1e-3 relative bound of the GPU parity tests
  bounds the input-dependent part of the output).
"""
import numpy as np
import pytest
import torch

from oracle.forward import NetOracle, rel_err
from oracle.torch_forward import TorchNet


def suite_and_weights(name):
    from paper_2304_09961_b200.executor import describe_suite, suite_weights
    d = describe_suite(name)
    return d, suite_weights(name, d)


def images(net, n, seed=1, first=0):
    from paper_2304_09961_b200.executor import make_image
    return np.stack([make_image(seed, first + i, net["in_H"], net["in_W"], net["in_C"]) for i in range(n)])


@pytest.mark.parametrize("suite", ["small_cnn", "googlenet", "resnet50", "mobilenet_v2"])
def test_numpy_oracle_matches_torch_functional(suite):
    d, w = suite_and_weights(suite)
    net = d["nets"][0]
    x = images(net, 2, seed=3)
    orc = NetOracle(d, 0, w)
    tn = TorchNet(d, 0, w, dtype=torch.float64)
    logits_t, _ = tn.forward(x)
    for i in range(2):
        blob = orc.forward(x[i])
        assert rel_err(orc.logits(blob), logits_t[i]) < 1e-5


@pytest.mark.parametrize("suite,min_classes", [("small_cnn", 10), ("googlenet", 50), ("resnet50", 50),
                                               ("mobilenet_v2", 50)])
def test_calibrated_outputs_are_input_dependent(suite, min_classes):
    d, w = suite_and_weights(suite)
    net = d["nets"][0]
    torch.set_num_threads(max(1, torch.get_num_threads()))
    x = images(net, 256, seed=1)
    logits, rms = TorchNet(d, 0, w, dtype=torch.float32).forward(x, record_rms=True)
    top1 = logits.argmax(1)
    assert len(set(top1.tolist())) >= min_classes
    assert np.bincount(top1).max() <= max(256 // 8, 3 * 256 // net["classes"])  # no class dominates
    bad = {k: v for k, v in rms.items() if not 0.1 <= v <= 10.0}
    assert not bad, bad
    # spread across inputs vs the common (input-independent) component
    spread = logits.std(axis=0).mean()
    common = np.abs(logits.mean(axis=0)).mean()
    assert spread > 1.5 * common, (spread, common)


def test_calibration_is_deterministic_and_tf32():
    from paper_2304_09961_b200.executor import describe_suite
    d, w = suite_and_weights("googlenet")
    _, w2 = suite_and_weights("googlenet")
    assert np.array_equal(w, w2)
    ops = [o for o in d["nets"][0]["ops"] if o["kind"] == "conv"]
    for o in ops[:5]:
        m = w[o["w_off"]:o["w_off"] + o["out"][2] * o["Kpad"]]
        assert np.all((m.view(np.uint32) & 0x1FFF) == 0)  # TF32-exact weights
    assert describe_suite("googlenet")["weights"] == w.size
