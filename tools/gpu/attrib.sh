# Attribution of conv time to pipeline roles via BS_CONV_DEBUG bits
# (1 skip converter TMEM stores, 2 skip lo MMA, 4 skip epilogue stores, 16 skip converter LDS, 32 skip epilogue).
for d in ${DEBUGS:-0 1 2 4 16 32 3 48 51}; do
  BS_CONV_DEBUG=$d timeout 120 python - <<PY
from tools.conv_bench import bench
r = [bench(90, H, Cin, N, k, pad, reps=20, res=rs) for (H, Cin, N, k, pad, rs) in [(28, 256, 288, 1, 0, 0), (56, 64, 256, 1, 0, 0), (56, 64, 256, 1, 0, 1), (28, 128, 512, 1, 0, 1), (14, 128, 256, 3, 1, 0), (7, 832, 384, 1, 0, 0)]]
print("debug=%-3d" % $d, "  ".join("%7.1f" % x for x in r), flush=True)
PY
done
