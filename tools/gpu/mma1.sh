mkdir -p gpurun_out/mma1
timeout 300 python -m pytest tests/test_kernels_gpu.py -x -q > gpurun_out/mma1/kt.log 2>&1; echo "rc=$?" >> gpurun_out/mma1/kt.log
for c in "90 28 96 128 3 1 1" "90 56 64 64 3 1 1" "90 56 64 192 3 1 1" "90 14 256 256 3 1 1" "90 224 4 64 7 2 3" "1 28 96 128 3 1 1"; do echo "$c: $(timeout 120 python tools/conv_case.py $c 20 2>&1 | tail -1)"; done > gpurun_out/mma1/cases.txt 2>&1
timeout 120 python tools/conv_trace_case.py 90 28 96 128 3 1 1 > gpurun_out/mma1/trace90_128.txt 2>&1
for a in "googlenet 90" "googlenet 1" "resnet50 90"; do timeout 300 python tools/b1_anatomy.py $a; done > gpurun_out/mma1/times.txt 2>&1
