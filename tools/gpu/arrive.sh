mkdir -p gpurun_out/arrive
timeout 300 python -m pytest tests/test_kernels_gpu.py -x -q > gpurun_out/arrive/kt.log 2>&1; echo "rc=$?" >> gpurun_out/arrive/kt.log
for c in "90 28 96 128 3 1 1" "90 56 64 64 3 1 1" "90 56 64 192 3 1 1" "90 14 256 256 3 1 1" "90 28 256 128 1 1 0" "90 224 4 64 7 2 3"; do echo "$c: $(timeout 120 python tools/conv_case.py $c 20 2>&1 | tail -1)"; done > gpurun_out/arrive/cases.txt 2>&1
for a in "googlenet 90" "resnet50 90" "googlenet 1"; do timeout 300 python tools/b1_anatomy.py $a; done >> gpurun_out/arrive/cases.txt 2>&1
