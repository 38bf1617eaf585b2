# per-layer launch lists at b=90 for the three activation paths
mkdir -p gpurun_out
for m in "win:BS_CONV_WIN=1" "gather:BS_CONV_WIN=0" ; do name=${m%%:*}; env=${m#*:}; env $env BS_CONV_LOG=1 timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/ll_$name.csv python tools/run_layers.py googlenet --batch 90 --reps 1 > gpurun_out/ll_$name.log 2>&1; done
