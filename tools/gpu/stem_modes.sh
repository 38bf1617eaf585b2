for env in "" "BS_CONV_TMA=1" "BS_CONV_WIN=1"; do
  env $env timeout 120 python -c "
from tools.conv_bench import bench
print('[$env] stem 7x7/2 224 4->64: %.1f us' % bench(90, 224, 4, 64, 7, 3, reps=10, stride=2), ' 3x3 56 64->192: %.1f us' % bench(90, 56, 64, 192, 3, 1, reps=10))"
done
