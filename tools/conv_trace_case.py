"""CTA-0 timeline of one conv shape (BS_CONV_TRACE=2: the second of two
back-to-back launches is traced).
    python tools/conv_trace_case.py nimg H Cin N k stride pad"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tests.test_kernels_gpu import run_conv  # noqa: E402

n, H, cin, N, k, s, pad = [int(x) for x in sys.argv[1:8]]
os.environ["BS_CONV_TRACE"] = "2"
print(f"== b={n} {H}x{H} {cin}->{N} {k}x{k}/{s}", flush=True)
print("err", run_conv(nimg=n, H=H, W=H, Cin=cin, N=N, KH=k, KW=k, stride=s, pad=pad, split=1, relu=1), flush=True)
