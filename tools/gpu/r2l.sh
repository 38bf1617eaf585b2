# 3x3 conv at b=90 (GoogLeNet i4-like and a 56x56 3x3): timings per precision + one full ncu capture each
mkdir -p gpurun_out/r2
python - > gpurun_out/r2/conv3x3_prec.txt 2>&1 <<'PY'
import sys; sys.path.insert(0, '.')
from tools.conv_bench import bench
for name, args in [("3x3 14x14 96->208", (90, 14, 96, 208, 3, 1)), ("3x3 28x28 128->192", (90, 28, 128, 192, 3, 1)),
                   ("3x3 56x56 64->192", (90, 56, 64, 192, 3, 1)), ("1x1 28x28 256->128", (90, 28, 256, 128, 1, 0)),
                   ("3x3 7x7 160->320", (90, 7, 160, 320, 3, 1))]:
    n, H, Cin, N, k, pad = args
    Ho = H
    flop = 2 * n * Ho * Ho * N * k * k * Cin
    for split in (1, 0, 2):
        us = bench(*args, reps=20, split=split)
        print(f"{name} prec={split}: {us:8.1f} us  {flop / us / 1e6:8.1f} TFLOP/s", flush=True)
PY
cat gpurun_out/r2/conv3x3_prec.txt
for sp in 1 2; do
timeout 400 ncu --set full --import-source on --clock-control none -k regex:conv_tc -s 1 -c 1 -o gpurun_out/r2/ncu_3x3_p$sp \
  python -c "
import sys; sys.path.insert(0, '.')
from tools.conv_bench import bench
print(bench(90, 28, 128, 192, 3, 1, reps=1, split=$sp))" > gpurun_out/r2/ncu_3x3_p$sp.log 2>&1
done
ls -la gpurun_out/r2/*.ncu-rep
