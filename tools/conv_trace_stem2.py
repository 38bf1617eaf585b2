"""CTA-0 timeline of the stem conv (7x7/2, 224 -> 112, Cin 4) at a batch:
per K tile (gather issue, landed, converted, MMA) and per unit (epilogue).
    BS_CONV_ROWWIN=0|1 python tools/conv_trace_stem2.py [nimg]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tests.test_kernels_gpu import run_conv  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8
os.environ["BS_CONV_TRACE"] = "2"
print(f"== stem b={n} rowwin={os.environ.get('BS_CONV_ROWWIN', '1')}", flush=True)
print("err", run_conv(nimg=n, H=224, W=224, Cin=4, N=64, KH=7, KW=7, stride=2, pad=3, split=1, relu=1), flush=True)
