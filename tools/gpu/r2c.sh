mkdir -p gpurun_out/r2
BS_CONV_LOG=1 timeout 300 python tools/conv_trace_b1.py > gpurun_out/r2/trace_b1.txt 2>&1
for ovh in 8 20 60; do BS_CONV_KS_OVH=$ovh timeout 300 python tools/span_bench.py googlenet:1,8 resnet50:1,8 > gpurun_out/r2/span_ovh$ovh.txt 2>&1; done
tail -n 5 gpurun_out/r2/span_ovh*.txt
