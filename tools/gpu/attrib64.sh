for d in 0 4 32; do
  BS_CONV_DEBUG=$d timeout 120 python - <<PY
from tools.conv_bench import bench
r = [bench(90, H, Cin, N, k, p, reps=20) for (H, Cin, N, k, p) in [(56, 64, 64, 1, 0), (56, 256, 64, 1, 0), (28, 192, 64, 1, 0), (56, 64, 128, 1, 0)]]
print("debug=%-3d" % $d, "  ".join("%7.1f" % x for x in r), flush=True)
PY
done
