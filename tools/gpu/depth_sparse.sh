# Steps in flight A/B with the sparse timed-region sampling (config 2).
mkdir -p gpurun_out/dep
for rep in 1 2; do for d in 3 4 5 6; do
  BENCH_DEPTH=$d timeout 900 python bench.py --cpu-forward 0 > gpurun_out/dep/c2_d${d}_r$rep.json 2> gpurun_out/dep/c2_d${d}_r$rep.err
done; done
