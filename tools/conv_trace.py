"""Prints the debug timeline of one conv launch (BS_CONV_TRACE)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["BS_CONV_TRACE"] = "1"
from tests.test_kernels_gpu import run_conv
for case in [dict(nimg=32, H=14, W=14, Cin=128, N=256, KH=3, KW=3, stride=1, pad=1)]:
    for split in (1, 0):
        print(case, "split", split, flush=True)
        print("err", run_conv(**case, split=split), flush=True)
