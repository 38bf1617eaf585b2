for d in 0 128; do
  BS_CONV_DEBUG=$d timeout 120 python -c "
from tools.conv_bench import bench
print('debug=$d stem: %.1f us' % bench(90, 224, 4, 64, 7, 3, reps=10, stride=2))"
done
DEBUGS="0 128" bash tools/gpu/attrib.sh
for d in 0 128; do
  for net in googlenet resnet50; do
    BS_CONV_DEBUG=$d timeout 200 python tools/run_layers.py $net --batch 90 --reps 5 > gpurun_out/l_${net}_$d.txt 2>&1
    python -c "
import re
t=[float(m) for m in re.findall(r'([0-9.]+)us', open('gpurun_out/l_${net}_$d.txt').read())]
print('debug=$d $net sum %.1f us' % sum(t))"
  done
done
