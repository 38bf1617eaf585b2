timeout 600 python -m pytest tests/test_kernels_gpu.py tests/test_executor_gpu.py -x -q 2>&1 | tail -1
for b in 90 32; do
for net in resnet50 googlenet; do
  timeout 200 python tools/run_layers.py $net --batch $b --reps 5 > gpurun_out/w2_$net.txt 2>&1
  python -c "
import re
t=[float(m) for m in re.findall(r'([0-9.]+)us', open('gpurun_out/w2_$net.txt').read())]
print('$net b=$b sum %.1f us' % sum(t))"
done
done
