# bf16x3 parity + latency tables for the precisions
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for pr in tf32x2 bf16x3; do timeout 300 python tools/profile_latency.py googlenet --precision $pr 2>&1 | tail -1; done
BS_CONV_LOG=1 timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/ll_bf16x3.csv python tools/run_layers.py googlenet --batch 90 --reps 1 --precision bf16x3 > gpurun_out/ll_bf16x3.log 2>&1
