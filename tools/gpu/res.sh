mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for net in resnet50 mobilenet_v2 googlenet; do timeout 300 python tools/profile_latency.py $net --batches 1,8,32,90 2>&1 | tail -1; done
BS_CONV_LOG=1 timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/ll_resnet50_res.csv python tools/run_layers.py resnet50 --batch 90 --reps 1 > gpurun_out/ll_resnet50_res.log 2>&1
