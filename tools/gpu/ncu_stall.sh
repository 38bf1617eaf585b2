mkdir -p gpurun_out/stall
# b=1 sequential long-K (one unit per CTA) and b=90 long-K / short-K shapes
BS_CONV_KS_MAX=1 timeout 300 ncu --set full --import-source on --clock-control none -k regex:conv_tc -s 3 -c 1 \
  -o gpurun_out/stall/b1_3x3_28 python tools/conv_case.py 1 28 96 128 3 1 1 5 > gpurun_out/stall/b1.log 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:conv_tc -s 3 -c 1 \
  -o gpurun_out/stall/b90_3x3_14 python tools/conv_case.py 90 14 96 208 3 1 1 5 > gpurun_out/stall/b90.log 2>&1
