# A/B of the conv kernel's super-stage pipeline (build/ab/ks2) vs the committed
# one (build/ab/base): kernel tests on the candidate, then shape and pass times.
mkdir -p gpurun_out/ks2
L=paper_2304_09961_b200/lib/libbs_exec.so
cp build/ab/ks2/libbs_exec.so $L
timeout 300 python -m pytest tests/test_kernels_gpu.py -x -q > gpurun_out/ks2/kt.log 2>&1; echo "rc=$?" >> gpurun_out/ks2/kt.log
for v in base ks2 base ks2; do
  cp build/ab/$v/libbs_exec.so $L
  for c in "90 28 96 128 3 1 1" "90 56 64 64 3 1 1" "90 56 64 192 3 1 1" "90 14 256 256 3 1 1" "90 28 256 128 1 1 0" "90 224 4 64 7 2 3"; do
    echo "$v $c: $(timeout 120 python tools/conv_case.py $c 20 2>&1 | tail -1)"; done
  for a in "googlenet 90" "resnet50 90" "googlenet 1"; do echo "$v $(timeout 300 python tools/b1_anatomy.py $a 2>&1 | tail -3 | tr '\n' ' ')"; done
done > gpurun_out/ks2/cases.txt 2>&1
cp build/ab/ks2/libbs_exec.so $L
