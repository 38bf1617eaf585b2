# conv micro-bench and per-layer b=90 launch lists for the activation paths
mkdir -p gpurun_out
for m in "gather:BS_CONV_TMA=0" "tma:BS_CONV_TMA=1"; do name=${m%%:*}; env=${m#*:}; echo "== $name"; env $env timeout 120 python tools/conv_bench.py 2>&1 | grep "b=90"; env $env BS_CONV_LOG=1 timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/ll_$name.csv python tools/run_layers.py googlenet --batch 90 --reps 1 > gpurun_out/ll_$name.log 2>&1; done
