mkdir -p gpurun_out/bn160
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/bn160/gputest.log 2>&1; echo "rc=$?" >> gpurun_out/bn160/gputest.log
for e in "BS_CONV_BN160=0" "BS_CONV_BN160=2"; do for c in "90 14 160 320 3 1 1" "90 7 160 320 3 1 1"; do
  echo "$e $c: $(env $e BS_CONV_BN192=0 timeout 120 python tools/conv_case.py $c 20 2>&1 | tail -1)"; done; done > gpurun_out/bn160/cases.txt 2>&1
for a in "googlenet 90" "googlenet 32" "googlenet 1" "mobilenet_v2 90"; do timeout 300 python tools/b1_anatomy.py $a; done > gpurun_out/bn160/times.txt 2>&1
timeout 900 python bench.py > gpurun_out/bn160/bench.json 2> gpurun_out/bn160/bench.err
