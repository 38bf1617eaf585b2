"""Batched CPU forward of the executor's networks with torch.nn.functional —
TEST INFRASTRUCTURE ONLY (a second, independent restatement of the layer math).

It pins oracle/layers.py (numpy, per image) to PyTorch's own CPU operators
(F.conv2d with zero padding, F.max_pool2d(ceil_mode=...), mean over H, W,
softmax) on the same exported network description and weights, and it is
fast enough (batched, oneDNN) to run the acceptance checks of SURVEY.md §7.4
over hundreds of inputs on the CPU: distinct top-1 classes and per-layer RMS.

PARITY UNPINNED w.r.t. the reference: batchsim has no forward pass
(proj/include/batchsim/simulator.hpp:702-721); see oracle/forward.py.

Only tests/, __graft_entry__.smoke() and bench.py's baseline legs may use it.
"""
from __future__ import annotations

import numpy as np
import torch
import torch.nn.functional as F


class TorchNet:
    def __init__(self, desc: dict, net: int, weights: np.ndarray, dtype=torch.float64, bf16_convs: bool = False):
        """bf16_convs: emulate the executor's BF16 precision -- every conv / FC
        multiplies bf16-rounded (nearest-even) activations and weights with
        high-precision accumulation; bias, residual, pools, depthwise convs and
        the stored activations stay fp32."""
        self.d = desc["nets"][net]
        self.w = torch.from_numpy(np.asarray(weights, np.float32))
        self.dtype = dtype
        self.bf16_convs = bf16_convs

    def _get(self, env, ref):
        t, coff, c = ref
        return env[t][:, coff:coff + c]

    def forward(self, images: np.ndarray, record_rms: bool = False):
        """images [N, H, W, C] (NHWC, C = padded input channels). Returns
        (logits [N, classes] float64 numpy, {op name: RMS of its output})."""
        d = self.d
        x = torch.from_numpy(np.ascontiguousarray(images)).to(self.dtype).permute(0, 3, 1, 2)
        n = x.shape[0]
        env = {}
        for i, T in enumerate(d["tensors"]):
            env[i] = torch.zeros((n, T["C"], T["H"], T["W"]), dtype=self.dtype)
        env[d["input"]][:] = x
        rms = {}
        for op in d["ops"]:
            kind = op["kind"]
            xin = self._get(env, op["in"])
            if kind == "conv":
                cin, cout, k = op["in"][2], op["out"][2], op["k"]
                K = k * k * cin
                w = self.w[op["w_off"]:op["w_off"] + cout * op["Kpad"]].reshape(cout, op["Kpad"])[:, :K]
                w = w.reshape(cout, k, k, cin).permute(0, 3, 1, 2).to(self.dtype)
                b = self.w[op["b_off"]:op["b_off"] + cout].to(self.dtype)
                if self.bf16_convs:
                    xin = xin.to(torch.bfloat16).to(self.dtype)
                    w = w.to(torch.bfloat16).to(self.dtype)
                y = F.conv2d(xin, w, b, stride=op["stride"], padding=op["pad"])
                if op["res"][0] >= 0:
                    y = y + self._get(env, op["res"])
            elif kind == "dwconv":
                c = op["in"][2]
                w = self.w[op["w_off"]:op["w_off"] + 9 * c].reshape(3, 3, c).permute(2, 0, 1)[:, None]
                b = self.w[op["b_off"]:op["b_off"] + c]
                y = F.conv2d(xin, w.to(self.dtype), b.to(self.dtype), stride=op["stride"], padding=1, groups=c)
            elif kind == "maxpool":
                y = F.max_pool2d(xin, op["k"], op["stride"], op["pad"], ceil_mode=bool(op["ceil"]))
            elif kind == "avgpool":
                y = xin.mean(dim=(2, 3), keepdim=True)
            elif kind == "softmax":
                y = torch.softmax(xin, dim=1)
            else:
                raise ValueError(kind)
            if op.get("relu") == 1:
                y = torch.clamp_min(y, 0)
            elif op.get("relu") == 2:
                y = torch.clamp(y, 0, 6)
            # every tensor is stored in fp32 between ops, like the executor's blobs
            y = y.to(torch.float32).to(self.dtype)
            t, coff, c = op["out"]
            env[t][:, coff:coff + c] = y
            if record_rms and kind != "softmax":
                rms[op["name"]] = float(torch.sqrt((y.double() ** 2).mean()))
        t, coff, c = d["logits"], 0, d["classes"]
        logits = env[t][:, coff:coff + c, 0, 0].double().numpy()
        return logits, rms
