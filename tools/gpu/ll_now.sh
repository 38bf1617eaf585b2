mkdir -p gpurun_out
for net in googlenet resnet50; do
BS_CONV_LOG=1 timeout 300 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/ll_${net}_now.csv python tools/run_layers.py $net --batch 90 --reps 1 > gpurun_out/ll_${net}_now.log 2>&1
done
