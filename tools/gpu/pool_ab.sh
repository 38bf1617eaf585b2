timeout 600 python -m pytest tests/test_kernels_gpu.py -x -q -k maxpool 2>&1 | tail -1
for blk in 22 24 44; do
  BS_POOL_BLOCK=$blk BS_CONV_LOG=1 timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/ll_pool_$blk.csv python tools/run_layers.py googlenet --batch 90 --reps 1 > gpurun_out/ll_pool_$blk.log 2>&1
  BS_POOL_BLOCK=$blk timeout 200 python tools/run_layers.py googlenet --batch 90 --reps 5 > gpurun_out/pl_$blk.txt 2>&1
  python -c "
import re
t=[float(m) for m in re.findall(r'([0-9.]+)us', open('gpurun_out/pl_$blk.txt').read())]
print('block=$blk googlenet b=90 sum %.1f us' % sum(t))"
done
