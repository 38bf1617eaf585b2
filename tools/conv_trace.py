"""Prints the debug timeline of one conv launch (BS_CONV_TRACE): per-CTA
start/setup/first-A/end and the first 48 K tiles of CTA 0.
    python tools/conv_trace.py [nimg]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["BS_CONV_TRACE"] = "1"
from tests.test_kernels_gpu import run_conv
nimg = int(sys.argv[1]) if len(sys.argv) > 1 else 32
for case in [dict(nimg=nimg, H=14, W=14, Cin=128, N=256, KH=3, KW=3, stride=1, pad=1)]:
    for split in (1,):
        print(case, "split", split, flush=True)
        print("err", run_conv(**case, split=split), flush=True)
