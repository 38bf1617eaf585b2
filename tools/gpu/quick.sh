# quick GPU check: kernel + executor parity, per-layer launch list at b=90, trace
mkdir -p gpurun_out
timeout 300 python -m pytest tests -m gpu -x -q > gpurun_out/quick_tests.log 2>&1; tail -2 gpurun_out/quick_tests.log
BS_CONV_LOG=1 timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/ll_b90_q.csv python tools/run_layers.py googlenet --batch 90 --reps 1 > gpurun_out/ll_b90_q.log 2>&1
timeout 300 python tools/profile_latency.py googlenet 2>&1 | tail -1
BS_CONV_TRACE=1 timeout 120 python tools/conv_trace.py > gpurun_out/trace.txt 2>&1
