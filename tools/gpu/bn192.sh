mkdir -p gpurun_out/bn192
timeout 300 python -m pytest tests/test_kernels_gpu.py -x -q > gpurun_out/bn192/kt.log 2>&1; echo "rc=$?" >> gpurun_out/bn192/kt.log
for bn in 0 2; do for c in "90 56 64 192 3 1 1" "90 28 128 192 3 1 1" "90 7 192 384 3 1 1" "90 14 96 208 3 1 1" "90 28 256 192 1 1 0"; do
  echo "bn192=$bn $c: $(BS_CONV_BN192=$bn timeout 120 python tools/conv_case.py $c 20 2>&1 | tail -1)"; done; done > gpurun_out/bn192/cases.txt 2>&1
for a in "googlenet 90" "googlenet 32" "googlenet 8"; do timeout 300 python tools/b1_anatomy.py $a; done > gpurun_out/bn192/times.txt 2>&1
