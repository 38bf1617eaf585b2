mkdir -p gpurun_out/g192
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/g192/gputest.log 2>&1; echo "rc=$?" >> gpurun_out/g192/gputest.log
for b in 0 2; do for a in "googlenet 90" "googlenet 32" "googlenet 8"; do BS_CONV_BN192=$b timeout 300 python tools/b1_anatomy.py $a | sed "s/^/bn192=$b /"; done; done > gpurun_out/g192/times.txt 2>&1
