mkdir -p gpurun_out/fc3
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/fc3/gputests.log 2>&1; echo "rc=$?" >> gpurun_out/fc3/gputests.log
for v in 0 1 0 1; do
  for a in "googlenet 1" "resnet50 1" "mobilenet_v2 1" "small_cnn 1" "resnet50 8"; do
    echo "gemv=$v $(BS_FC_GEMV=$v timeout 300 python tools/b1_anatomy.py $a 2>&1 | tail -3 | tr '\n' ' ')"; done
done > gpurun_out/fc3/passes.txt 2>&1
timeout 600 ncu --set full --clock-control none -k regex:fc_gemv -s 2 -c 1 -o gpurun_out/fc3/fc_gemv_resnet50_b1 python tools/b1_anatomy.py resnet50 1 > /dev/null 2>&1
