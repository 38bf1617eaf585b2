mkdir -p gpurun_out/mc
timeout 300 python -m pytest tests/test_kernels_gpu.py -x -q > gpurun_out/mc/kt.log 2>&1
echo "kt rc=$?" >> gpurun_out/mc/kt.log
for mc in 0 1; do
  for a in "googlenet 90" "resnet50 90" "googlenet 32"; do BS_CONV_MC=$mc timeout 300 python tools/b1_anatomy.py $a | sed "s/^/mc=$mc /"; done
done > gpurun_out/mc/times.txt 2>&1
