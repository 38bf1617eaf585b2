mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 300 python tools/profile_latency.py mobilenet_v2 --batches 1,8,32,90 2>&1 | tail -1
BS_CONV_LOG=1 timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/ll_mobilenet_v2_dw.csv python tools/run_layers.py mobilenet_v2 --batch 90 --reps 1 > gpurun_out/ll_mobilenet_v2_dw.log 2>&1
