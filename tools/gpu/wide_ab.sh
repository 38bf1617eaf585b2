for w in 1 2; do
  BS_CONV_BN256=$w DEBUGS="0" bash tools/gpu/attrib_res.sh | sed "s/^/bn256=$w /"
  for net in resnet50 googlenet; do
    BS_CONV_BN256=$w BS_CONV_LOG=1 timeout 200 python tools/run_layers.py $net --batch 90 --reps 3 > gpurun_out/w_${net}_$w.txt 2>&1
    python -c "
import re
t=[float(m) for m in re.findall(r'([0-9.]+)us', open('gpurun_out/w_${net}_$w.txt').read())]
print('bn256=$w $net b=90 sum %.1f us' % sum(t))"
  done
done
