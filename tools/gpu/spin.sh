mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 120 python tools/conv_bench.py 2>&1 | grep -E "b=90|b= 8"
for net in googlenet mobilenet_v2; do timeout 120 python tools/run_layers.py $net --batch 90 --from 1 --to 3 --reps 5; done
timeout 300 python tools/profile_latency.py googlenet 2>&1 | tail -1
timeout 300 python tools/profile_latency.py mobilenet_v2 --batches 1,8,32,90 2>&1 | tail -1
timeout 300 python tools/profile_latency.py resnet50 --batches 1,8,32,90 2>&1 | tail -1
