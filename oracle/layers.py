"""CPU fp32 NHWC layer math — TEST INFRASTRUCTURE ONLY (the layer-output oracle).

PARITY UNPINNED w.r.t. the reference: batchsim (arXiv 2304.09961) has no
forward pass at all — a batched step is a cost-table lookup
(proj/include/batchsim/simulator.hpp:702-721). These are the
textbook definitions of the ops the north_star's networks use (conv with
zero padding, max-pool with ceil mode, global average pool, FC, softmax),
written independently of the CUDA path so they can check it.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may use
this module.
"""
from __future__ import annotations

import numpy as np


def round_bf16(x: np.ndarray) -> np.ndarray:
    """Round fp32 to bf16 (8-bit mantissa), nearest-even, kept as fp32 -- the
    rounding of PTX cvt.rn.bf16x2.f32 / __float2bfloat16_rn (finite x)."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    u = x.view(np.uint32).astype(np.uint64)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000).astype(np.uint32)
    return r.view(np.float32)


def round_tf32(x: np.ndarray) -> np.ndarray:
    """Round fp32 to TF32 (10-bit mantissa), nearest, ties away from zero —
    the rounding of PTX cvt.rna.tf32.f32."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    u = x.view(np.uint32).astype(np.uint64)
    exp_all_ones = (u & 0x7F800000) == 0x7F800000
    r = ((u + 0x1000) & 0xFFFFE000).astype(np.uint32)
    r = np.where(exp_all_ones, u.astype(np.uint32), r)
    return r.view(np.float32)


def conv2d_nhwc(x: np.ndarray, w: np.ndarray, b: np.ndarray | None, stride: int, pad: int,
                acc=np.float64) -> np.ndarray:
    """x [N,H,W,C], w [Cout,KH,KW,C] -> [N,Ho,Wo,Cout]; zero padding."""
    n, h, wd, c = x.shape
    cout, kh, kw, c2 = w.shape
    assert c == c2
    ho = (h + 2 * pad - kh) // stride + 1
    wo = (wd + 2 * pad - kw) // stride + 1
    xp = np.zeros((n, h + 2 * pad, wd + 2 * pad, c), dtype=acc)
    xp[:, pad:pad + h, pad:pad + wd, :] = x
    cols = np.empty((n, ho, wo, kh, kw, c), dtype=acc)
    for i in range(kh):
        for j in range(kw):
            cols[:, :, :, i, j, :] = xp[:, i:i + stride * ho:stride, j:j + stride * wo:stride, :]
    y = cols.reshape(n * ho * wo, kh * kw * c) @ w.reshape(cout, -1).astype(acc).T
    if b is not None:
        y = y + b.astype(acc)
    return y.reshape(n, ho, wo, cout)


def depthwise3x3_nhwc(x: np.ndarray, w: np.ndarray, b: np.ndarray | None, stride: int,
                      acc=np.float64) -> np.ndarray:
    """x [N,H,W,C], w [C,3,3] (pad 1)."""
    n, h, wd, c = x.shape
    ho = (h + 2 - 3) // stride + 1
    wo = (wd + 2 - 3) // stride + 1
    xp = np.zeros((n, h + 2, wd + 2, c), dtype=acc)
    xp[:, 1:1 + h, 1:1 + wd, :] = x
    y = np.zeros((n, ho, wo, c), dtype=acc)
    for i in range(3):
        for j in range(3):
            y += xp[:, i:i + stride * ho:stride, j:j + stride * wo:stride, :] * w[:, i, j].astype(acc)
    if b is not None:
        y += b.astype(acc)
    return y


def maxpool_nhwc(x: np.ndarray, k: int, stride: int, pad: int, ceil: bool) -> np.ndarray:
    n, h, wd, c = x.shape

    def out(sz):
        num = sz + 2 * pad - k
        o = (-(-num // stride) if ceil else num // stride) + 1
        # PyTorch rule: the last window must start inside the (left-padded) input.
        if ceil and (o - 1) * stride >= sz + pad:
            o -= 1
        return o

    ho, wo = out(h), out(wd)
    y = np.full((n, ho, wo, c), -np.inf, dtype=x.dtype)
    for i in range(ho):
        for j in range(wo):
            h0, w0 = i * stride - pad, j * stride - pad
            hs, ws = max(h0, 0), max(w0, 0)
            he, we = min(h0 + k, h), min(w0 + k, wd)
            y[:, i, j, :] = x[:, hs:he, ws:we, :].max(axis=(1, 2))
    return y


def global_avgpool_nhwc(x: np.ndarray, acc=np.float64) -> np.ndarray:
    return x.astype(acc).mean(axis=(1, 2))


def softmax(x: np.ndarray) -> np.ndarray:
    z = x - x.max(axis=-1, keepdims=True)
    e = np.exp(z)
    return e / e.sum(axis=-1, keepdims=True)
