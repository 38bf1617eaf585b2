# Small-batch anatomy: pass times with/without PDL, and a warm ncu launch list.
mkdir -p gpurun_out/b1
for pdl in 0 1; do
  for a in "small_cnn 1" "googlenet 1" "googlenet 8" "resnet50 1"; do
    BS_PDL=$pdl timeout 300 python tools/b1_anatomy.py $a
  done
done > gpurun_out/b1/times.txt 2>&1
timeout 600 ncu --cache-control none --clock-control none --metrics gpu__time_duration.sum --csv \
  --log-file gpurun_out/b1/googlenet_b1_warm.csv python tools/b1_anatomy.py googlenet 1 ncu > /dev/null 2>&1
timeout 600 ncu --cache-control none --clock-control none --metrics gpu__time_duration.sum --csv \
  --log-file gpurun_out/b1/small_cnn_b1_warm.csv python tools/b1_anatomy.py small_cnn 1 ncu > /dev/null 2>&1
cuobjdump -res-usage paper_2304_09961_b200/lib/libbs_exec.so > gpurun_out/b1/resusage.txt 2>&1
