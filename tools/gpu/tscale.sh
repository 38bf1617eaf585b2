mkdir -p gpurun_out/tscale
for t in 1 0; do
  for r in 1 2; do BS_TABLE_SCALE=$t timeout 900 python bench.py --steps 3 --cpu-forward 0 > gpurun_out/tscale/c2_s${t}_$r.json 2>/dev/null; done
  BS_TABLE_SCALE=$t timeout 900 python bench.py --config 4 --steps 3 --cpu-forward 0 > gpurun_out/tscale/c4_s$t.json 2>/dev/null
  BS_TABLE_SCALE=$t timeout 900 python bench.py --config 1 --steps 3 --cpu-forward 0 > gpurun_out/tscale/c1_s$t.json 2>/dev/null
done
