import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tools.conv_bench import bench
print(bench(1, 14, 128, 256, 3, 1, reps=5, split=int(sys.argv[1]) if len(sys.argv) > 1 else 1))
