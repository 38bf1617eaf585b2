mkdir -p gpurun_out
for net in resnet50 mobilenet_v2; do
  timeout 300 python tools/profile_latency.py $net --batches 1,8,32,90 2>&1 | tail -1
  BS_CONV_LOG=1 timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/ll_$net.csv python tools/run_layers.py $net --batch 90 --reps 1 > gpurun_out/ll_$net.log 2>&1
done
