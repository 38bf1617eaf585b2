"""BS_CONV_TRACE timeline of a short-K 1x1 conv (epilogue-heavy): 28x28, 256 -> 288 at batch n."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["BS_CONV_TRACE"] = "1"
from tests.test_kernels_gpu import run_conv
n = int(sys.argv[1]) if len(sys.argv) > 1 else 90
print("err", run_conv(nimg=n, H=28, W=28, Cin=256, N=288, KH=1, KW=1, stride=1, pad=0, split=1), flush=True)
