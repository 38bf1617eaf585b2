mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
for pdl in 1 0; do
 for b in 90 8; do
  for net in googlenet resnet50; do
    BS_PDL=$pdl timeout 200 python tools/run_layers.py $net --batch $b --reps 5 > gpurun_out/p_$net.txt 2>&1
    python -c "
import re
t=[float(m) for m in re.findall(r'([0-9.]+)us', open('gpurun_out/p_$net.txt').read())]
print('pdl=$pdl b=$b $net sum %.1f us' % sum(t))"
  done
 done
done
