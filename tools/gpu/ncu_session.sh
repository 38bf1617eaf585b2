# ncu --set full of this round's reworked paths: tap-row stem, short-K 1x1 epilogue, residual 1x1.
mkdir -p gpurun_out
for spec in "stem:90,224,4,64,7,3,0,2" "1x1_56:90,56,64,256,1,0,0,1" "1x1_56_res:90,56,64,256,1,0,1,1"; do
  name=${spec%%:*}; args=${spec#*:}
  IFS=, read n H Cin N k pad res stride <<< "$args"
  timeout 400 ncu --set full --import-source on --clock-control none -k regex:conv_tc -c 1 -o gpurun_out/ncu_s3_$name \
    python -c "
import sys; sys.path.insert(0, '.')
from tools.conv_bench import bench
print(bench($n, $H, $Cin, $N, $k, $pad, reps=1, res=bool($res), stride=$stride))" > gpurun_out/ncu_s3_$name.log 2>&1
  echo "$name rc=$?"
done
