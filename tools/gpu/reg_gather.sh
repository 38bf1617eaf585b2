# A/B of the register-staged A gather (BS_REG_GATHER=1) vs cp.async (0):
# kernel parity with the candidate, then conv shape and whole-pass times.
mkdir -p gpurun_out/rg
BS_REG_GATHER=1 timeout 600 python -m pytest tests/test_kernels_gpu.py -x -q > gpurun_out/rg/kt.log 2>&1; echo "rc=$?" >> gpurun_out/rg/kt.log
BS_REG_GATHER=1 timeout 600 python -m pytest tests/test_executor_gpu.py -x -q -k "ragged or full_batch or mobilenet or riders_and" > gpurun_out/rg/ex.log 2>&1; echo "rc=$?" >> gpurun_out/rg/ex.log
for v in 0 1 0 1; do
  for c in "90 28 96 128 3 1 1" "90 56 64 64 3 1 1" "90 56 64 192 3 1 1" "90 14 256 256 3 1 1" "90 28 256 128 1 1 0" "8 28 96 128 3 1 1"; do
    echo "rg=$v $c: $(BS_REG_GATHER=$v timeout 120 python tools/conv_case.py $c 20 2>&1 | tail -1)"; done
  for a in "googlenet 90" "resnet50 90" "googlenet 8" "googlenet 1"; do echo "rg=$v $(BS_REG_GATHER=$v timeout 300 python tools/b1_anatomy.py $a 2>&1 | tail -3 | tr '\n' ' ')"; done
done > gpurun_out/rg/cases.txt 2>&1
