mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for g in 1 0; do
 for b in 90 32 8; do
  for net in googlenet resnet50; do
    BS_CONV_GROUP=$g timeout 200 python tools/run_layers.py $net --batch $b --reps 5 > gpurun_out/g_$net.txt 2>&1
    python -c "
import re
t=[float(m) for m in re.findall(r'([0-9.]+)us', open('gpurun_out/g_$net.txt').read())]
print('group=$g b=$b $net sum %.1f us' % sum(t))"
  done
 done
done
