timeout 600 python -m pytest tests/test_kernels_gpu.py tests/test_executor_gpu.py -x -q 2>&1 | tail -1
DEBUGS="0 256" bash tools/gpu/attrib_res.sh
for d in 0 256; do
  BS_CONV_DEBUG=$d timeout 200 python tools/run_layers.py resnet50 --batch 90 --reps 5 > gpurun_out/r_$d.txt 2>&1
  python -c "
import re
t=[float(m) for m in re.findall(r'([0-9.]+)us', open('gpurun_out/r_$d.txt').read())]
print('debug=$d resnet50 b=90 sum %.1f us' % sum(t))"
done
