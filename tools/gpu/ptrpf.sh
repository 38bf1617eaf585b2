timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
bash tools/gpu/attrib64.sh | head -1
DEBUGS=0 bash tools/gpu/attrib.sh
DEBUGS=0 bash tools/gpu/attrib_res.sh
for net in googlenet resnet50; do
  timeout 200 python tools/run_layers.py $net --batch 90 --reps 5 > gpurun_out/pp_$net.txt 2>&1
  python -c "
import re
t=[float(m) for m in re.findall(r'([0-9.]+)us', open('gpurun_out/pp_$net.txt').read())]
print('$net b=90 sum %.1f us' % sum(t))"
done
