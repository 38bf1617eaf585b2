"""Small-batch conv anatomy: BS_CONV_TRACE timeline (CTA start / setup /
first A / end) plus the back-to-back launch time of the same conv.
    python tools/conv_trace_b1.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tests.test_kernels_gpu import run_conv  # noqa: E402
from tools.conv_bench import bench  # noqa: E402

cases = [  # (name, nimg, H, Cin, N, k, stride, pad)
    ("smallcnn conv1 32x32 4->32 3x3", 1, 32, 4, 32, 3, 1, 1),
    ("smallcnn conv2 32x32 32->64 3x3/2", 1, 32, 32, 64, 3, 2, 1),
    ("smallcnn conv3 16x16 64->128 3x3/2", 1, 16, 64, 128, 3, 2, 1),
    ("inception 1x1 14x14 480->192", 1, 14, 480, 192, 1, 1, 0),
    ("inception 3x3 14x14 96->208", 1, 14, 96, 208, 3, 1, 1),
    ("1x1 7x7 832->384", 1, 7, 832, 384, 1, 1, 0),
]
for name, n, H, cin, N, k, s, pad in cases:
    os.environ["BS_CONV_TRACE"] = "1"
    print(f"== {name} b={n}", flush=True)
    err = run_conv(nimg=n, H=H, W=H, Cin=cin, N=N, KH=k, KW=k, stride=s, pad=pad, split=1)
    os.environ.pop("BS_CONV_TRACE")
    print(f"err {err:.2e}  back-to-back launch {bench(n, H, cin, N, k, pad, stride=s, reps=200):.2f} us", flush=True)
