"""BS_CONV_TRACE timeline of a small conv (one unit per CTA): 3x3 14x14 16 -> 48 at batch n."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["BS_CONV_TRACE"] = "1"
from tests.test_kernels_gpu import run_conv
from tools.conv_bench import bench
n = int(sys.argv[1]) if len(sys.argv) > 1 else 90
print("err", run_conv(nimg=n, H=14, W=14, Cin=16, N=48, KH=3, KW=3, stride=1, pad=1, split=1), flush=True)
os.environ.pop("BS_CONV_TRACE")
print("back-to-back launch: %.1f us" % bench(n, 14, 16, 48, 3, 1, reps=50), flush=True)
