timeout 600 python -m pytest tests/test_kernels_gpu.py tests/test_executor_gpu.py -x -q 2>&1 | tail -1
BS_CONV_NMINOR=1 timeout 600 python -m pytest tests/test_kernels_gpu.py tests/test_executor_gpu.py -x -q 2>&1 | tail -1
for m in 0 1; do
  BS_CONV_NMINOR=$m DEBUGS=0 bash tools/gpu/attrib_res.sh | sed "s/^/nminor=$m /"
  for net in googlenet resnet50; do
    BS_CONV_NMINOR=$m timeout 200 python tools/run_layers.py $net --batch 90 --reps 5 > gpurun_out/nm_$net.txt 2>&1
    python -c "
import re
t=[float(x) for x in re.findall(r'([0-9.]+)us', open('gpurun_out/nm_$net.txt').read())]
print('nminor=$m $net b=90 sum %.1f us' % sum(t))"
  done
done
