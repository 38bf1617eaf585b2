mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_kernels_gpu.py -x -q 2>&1 | tail -2
for mode in 0 1; do BS_CONV_TMA=$mode BS_CONV_LOG=1 timeout 300 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/ll_b90_t$mode.csv python tools/run_layers.py googlenet --batch 90 --reps 1 > gpurun_out/ll_b90_t$mode.log 2>&1; done
