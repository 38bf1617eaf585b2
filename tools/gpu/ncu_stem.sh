mkdir -p gpurun_out
timeout 400 ncu --set full --import-source on --clock-control none -k regex:conv_tc -c 1 -o gpurun_out/ncu_stem \
  python -c "
import sys; sys.path.insert(0, '.')
from tools.conv_bench import bench
print(bench(90, 224, 4, 64, 7, 3, reps=1, stride=2))" > gpurun_out/ncu_stem.log 2>&1
tail -2 gpurun_out/ncu_stem.log
