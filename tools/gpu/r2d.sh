mkdir -p gpurun_out/r2
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r2/pytest_cluster.txt 2>&1; tail -n 15 gpurun_out/r2/pytest_cluster.txt
for ovh in 2 4 8 16; do echo "ovh $ovh"; BS_CONV_KS_OVH=$ovh timeout 300 python tools/span_bench.py small_cnn:1,10 googlenet:1,8,32 resnet50:1,8 mobilenet_v2:1,8; done > gpurun_out/r2/span_cluster.txt 2>&1
cat gpurun_out/r2/span_cluster.txt
BS_CONV_LOG=1 timeout 300 python tools/conv_trace_b1.py 2>&1 | grep -v "^conv M" > gpurun_out/r2/trace_b1_cluster.txt
