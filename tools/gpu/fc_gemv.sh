# Small-batch FC as a weight-streaming GEMV: GPU parity suite, then whole-pass
# A/B (BS_FC_GEMV=0 keeps conv_tc for the FC) at b = 1 / 4 / 8.
mkdir -p gpurun_out/fc
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/fc/gputests.log 2>&1; echo "rc=$?" >> gpurun_out/fc/gputests.log
for v in 0 1 0 1; do
  for a in "googlenet 1" "googlenet 8" "resnet50 1" "mobilenet_v2 1" "small_cnn 1"; do
    echo "gemv=$v $(BS_FC_GEMV=$v timeout 300 python tools/b1_anatomy.py $a 2>&1 | tail -3 | tr '\n' ' ')"; done
done > gpurun_out/fc/passes.txt 2>&1
