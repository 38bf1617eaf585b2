"""One 3x3 14x14 128->256 conv at batch 90 through the kernel hook (for ncu)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tools.conv_bench import bench
print(bench(90, 14, 128, 256, 3, 1, reps=3, split=1))
