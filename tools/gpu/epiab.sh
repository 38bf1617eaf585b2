# Epilogue timing: conv shapes at b=90 through the kernel hook + per-layer executor sums.
mkdir -p gpurun_out
for d in ${DEBUGS:-0}; do
  echo "== BS_CONV_DEBUG=$d"
  BS_CONV_DEBUG=$d timeout 120 python - <<'PY'
from tools.conv_bench import bench
for (H, Cin, N, k, pad) in [(28, 256, 288, 1, 0), (14, 128, 256, 3, 1), (7, 832, 384, 1, 0), (56, 64, 256, 1, 0), (56, 64, 64, 3, 1)]:
    print(f"b=90 {k}x{k} {H}x{H} {Cin}->{N}: {bench(90, H, Cin, N, k, pad, reps=20):7.1f} us", flush=True)
PY
  for net in googlenet resnet50; do
    BS_CONV_DEBUG=$d timeout 200 python tools/run_layers.py $net --batch 90 --reps 5 > gpurun_out/layers_${net}_d$d.txt 2>&1
    python -c "
import re,sys
t=[float(m) for m in re.findall(r'([0-9.]+)us', open('gpurun_out/layers_${net}_d$d.txt').read())]
print('$net', 'layers', len(t), 'sum %.1f us' % sum(t))"
  done
done
[ -n "$PARITY" ] && timeout 600 python -m pytest tests/test_kernels_gpu.py tests/test_executor_gpu.py -x -q 2>&1 | tail -2
true
