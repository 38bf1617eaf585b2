mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
timeout 600 compute-sanitizer --tool memcheck --print-limit 5 python -m pytest tests/test_kernels_gpu.py -x -q -k "matches_oracle or tap_rows" 2>&1 | tail -4
BS_CONV_TAPROW=1 timeout 120 python -c "
from tools.conv_bench import bench
print('stem 7x7/2 224 4->64: %.1f us' % bench(90, 224, 4, 64, 7, 3, reps=10, stride=2))"
DEBUGS="0" bash tools/gpu/attrib.sh
