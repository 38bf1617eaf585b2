"""Back-to-back launches of one b=90 conv for ~N seconds (clock / power sampling)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tools.conv_bench import bench
t = time.time()
while time.time() - t < float(sys.argv[1] if len(sys.argv) > 1 else 5):
    us = bench(90, 14, 128, 256, 3, 1, reps=400, split=1)
print("last us/launch", us)
