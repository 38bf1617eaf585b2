mkdir -p gpurun_out/g192
for r in 1 2; do for g in 0 1; do for a in "googlenet 90" "googlenet 32" "googlenet 8"; do BS_CONV_G192=$g timeout 300 python tools/b1_anatomy.py $a | sed "s/^/g192=$g /"; done; done; done > gpurun_out/g192/times2.txt 2>&1
