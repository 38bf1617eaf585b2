mkdir -p gpurun_out
for b in 1 8; do
  timeout 200 python tools/run_layers.py googlenet --batch $b --reps 20 > gpurun_out/sb_$b.txt 2>&1
  python -c "
import re
t=[float(m) for m in re.findall(r'([0-9.]+)us', open('gpurun_out/sb_$b.txt').read())]
print('b=$b layer-event sum %.1f us' % sum(t))"
  BS_CONV_LOG=1 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ll_sb_$b.csv python tools/run_layers.py googlenet --batch $b --reps 1 > gpurun_out/ll_sb_$b.log 2>&1
done
