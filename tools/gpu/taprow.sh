mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for tr in 1 0; do
  BS_CONV_TAPROW=$tr timeout 120 python -c "
from tools.conv_bench import bench
print('taprow=$tr stem 7x7/2 224 4->64: %.1f us' % bench(90, 224, 4, 64, 7, 3, reps=10, stride=2))"
  BS_CONV_TAPROW=$tr timeout 200 python tools/run_layers.py googlenet --batch 90 --from 1 --to 1 --reps 5
  BS_CONV_TAPROW=$tr timeout 200 python tools/run_layers.py resnet50 --batch 90 --from 1 --to 1 --reps 5
done
