"""Per-K-tile timeline of CTA 0 for b=1 convs with long K loops (warm L2):
which ring paces a single CTA's K loop (A gather, conversion, B TMA, MMA)?
    BS_CONV_KS_MAX=1 python tools/conv_trace_seq.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tests.test_kernels_gpu import run_conv  # noqa: E402

cases = [  # (name, nimg, H, Cin, N, k, stride, pad)
    ("3x3 28x28 96->128", 1, 28, 96, 128, 3, 1, 1),
    ("3x3 14x14 112->224 (N>128)", 1, 14, 112, 224, 3, 1, 1),
    ("1x1 7x7 832->384", 1, 7, 832, 384, 1, 1, 0),
    ("3x3 16x16 64->128 /2", 1, 16, 64, 128, 3, 2, 1),
]
for name, n, H, cin, N, k, s, pad in cases:
    os.environ["BS_CONV_TRACE"] = os.environ.get("TRACE_MODE", "1")
    print(f"== {name} b={n}", flush=True)
    err = run_conv(nimg=n, H=H, W=H, Cin=cin, N=N, KH=k, KW=k, stride=s, pad=pad, split=int(os.environ.get("PREC", "1")))
    os.environ.pop("BS_CONV_TRACE")
    print(f"err {err:.2e}", flush=True)
