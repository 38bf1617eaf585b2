mkdir -p gpurun_out/clk
for r in 1 2; do for c in host device; do
  BENCH_COMPLETION_CLOCK=$c timeout 900 python bench.py --steps 3 --cpu-forward 0 > gpurun_out/clk/c2_${c}_$r.json 2>/dev/null
done; done
