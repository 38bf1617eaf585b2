# Parity + small conv timeline + stem + network layer sums at b=90.
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
timeout 120 python tools/conv_trace_small.py 90 2>&1 | grep -E "it +[0-4] |back-to-back|cta   0"
timeout 120 python -c "
from tools.conv_bench import bench
print('stem: %.1f us' % bench(90, 224, 4, 64, 7, 3, reps=10, stride=2))"
for net in googlenet resnet50 mobilenet_v2; do
  timeout 200 python tools/run_layers.py $net --batch 90 --reps 5 > gpurun_out/q_$net.txt 2>&1
  python -c "
import re
t=[float(m) for m in re.findall(r'([0-9.]+)us', open('gpurun_out/q_$net.txt').read())]
print('$net sum %.1f us' % sum(t))"
done
