mkdir -p gpurun_out/his
python -m pytest tests/test_kernels_gpu.py -x -q > gpurun_out/his/kt.log 2>&1
BS_CONV_KS_MAX=1 python tools/conv_trace_seq.py > gpurun_out/his/trace_seq.txt 2>&1
for a in "googlenet 90" "googlenet 8" "googlenet 1" "resnet50 90"; do timeout 300 python tools/b1_anatomy.py $a; done > gpurun_out/his/times.txt 2>&1
