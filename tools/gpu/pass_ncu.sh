# warm per-kernel list of one whole-network pass (after the autotune), one net/batch per arg pair
mkdir -p gpurun_out/pass
while [ $# -gt 1 ]; do
  timeout 600 ncu --profile-from-start off --cache-control none --clock-control none \
    --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active \
    --csv --log-file gpurun_out/pass/$1_b$2.csv python tools/b1_anatomy.py $1 $2 ncu > /dev/null 2>&1
  shift 2
done
