# ResNet residual 1x1 shapes at b=90: debug 0 full, 4 skip stores, 32 skip epilogue, 64 no residual prefetch.
for d in ${DEBUGS:-0 4 32 64}; do
  BS_CONV_DEBUG=$d timeout 120 python - <<PY
from tools.conv_bench import bench
r = [bench(90, H, Cin, N, 1, 0, reps=20, res=rs) for (H, Cin, N, rs) in [(14, 256, 1024, 1), (14, 256, 1024, 0), (56, 64, 256, 1), (28, 128, 512, 1)]]
print("debug=%-3d" % $d, "  ".join("%7.1f" % x for x in r), flush=True)
PY
done
