"""Prints the debug timeline of one conv launch (BS_CONV_TRACE)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["BS_CONV_TRACE"] = "1"
from tests.test_kernels_gpu import run_conv
for case in [dict(nimg=1, H=7, W=7, Cin=832, N=384, KH=1, KW=1, stride=1, pad=0),
             dict(nimg=90, H=7, W=7, Cin=192, N=384, KH=3, KW=3, stride=1, pad=1),
             dict(nimg=8, H=1, W=1, Cin=1024, N=1000, KH=1, KW=1, stride=1, pad=0)]:
    for split in (0, 1):
        print(case, "split", split, flush=True)
        err = run_conv(**case, split=split)
        print("err", err, flush=True)
