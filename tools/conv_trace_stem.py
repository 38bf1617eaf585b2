"""BS_CONV_TRACE timeline of the GoogLeNet/ResNet stem (7x7/2, Cin 4, N 64) at batch n."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["BS_CONV_TRACE"] = "1"
from tests.test_kernels_gpu import run_conv
n = int(sys.argv[1]) if len(sys.argv) > 1 else 16
print("err", run_conv(nimg=n, H=224, W=224, Cin=4, N=64, KH=7, KW=7, stride=2, pad=3, split=1), flush=True)
