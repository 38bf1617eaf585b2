mkdir -p gpurun_out
timeout 400 ncu --set full --import-source on --clock-control none -k regex:conv_tc -c 1 -o gpurun_out/ncu_1x1_56 \
  python -c "
import sys; sys.path.insert(0, '.')
from tools.conv_bench import bench
print(bench(90, 56, 64, 256, 1, 0, reps=1))" > gpurun_out/ncu_1x1_56.log 2>&1
tail -3 gpurun_out/ncu_1x1_56.log
