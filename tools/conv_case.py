"""One conv shape through the kernel hook, `reps` back-to-back launches
(for ncu captures of a single shape).
    python tools/conv_case.py nimg H Cin N k stride pad [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tools.conv_bench import bench  # noqa: E402

a = [int(x) for x in sys.argv[1:]]
nimg, H, Cin, N, k, s, pad = a[:7]
reps = a[7] if len(a) > 7 else 5
print(f"{bench(nimg, H, Cin, N, k, pad, stride=s, reps=reps):.2f} us per launch")
