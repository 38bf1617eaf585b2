mkdir -p gpurun_out/b1
for pdl in 0 1; do
  for a in "small_cnn 1" "googlenet 1" "googlenet 8" "resnet50 1" "googlenet 90"; do
    BS_PDL=$pdl timeout 300 python tools/b1_anatomy.py $a
  done
done > gpurun_out/b1/times_${1:-x}.txt 2>&1
