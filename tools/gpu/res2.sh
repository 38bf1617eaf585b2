mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
BS_CONV_LOG=1 timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/ll_g_res2.csv python tools/run_layers.py googlenet --batch 90 --reps 1 > gpurun_out/ll_g_res2.log 2>&1
BS_CONV_LOG=1 timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/ll_r_res2.csv python tools/run_layers.py resnet50 --batch 90 --reps 1 > gpurun_out/ll_r_res2.log 2>&1
