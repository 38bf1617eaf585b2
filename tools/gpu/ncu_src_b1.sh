mkdir -p gpurun_out/stall
BS_CONV_KS_MAX=1 timeout 300 ncu --section SourceCounters --section WarpStateStats --warp-sampling-interval 0 --cache-control none \
  --import-source on --clock-control none -k regex:conv_tc -s 3 -c 1 \
  -o gpurun_out/stall/b1_src python tools/conv_case.py 1 28 96 128 3 1 1 5 > gpurun_out/stall/b1src.log 2>&1
timeout 300 ncu --section SourceCounters --section WarpStateStats --warp-sampling-interval 1 --cache-control none \
  --import-source on --clock-control none -k regex:conv_tc -s 3 -c 1 \
  -o gpurun_out/stall/b90_src python tools/conv_case.py 90 28 96 128 3 1 1 5 > gpurun_out/stall/b90src.log 2>&1
