mkdir -p gpurun_out/depth2
for cfg in 3 4 5 1; do for d in 2 3; do
  BENCH_DEPTH=$d timeout 900 python bench.py --config $cfg --steps 3 --cpu-forward 0 > gpurun_out/depth2/c${cfg}_d$d.json 2>/dev/null
done; done
