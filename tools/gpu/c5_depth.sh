mkdir -p gpurun_out/c5d
for rep in 1 2; do for d in 2 4; do
  BENCH_DEPTH=$d timeout 900 python bench.py --config 5 > gpurun_out/c5d/c5_d${d}_r$rep.json 2> gpurun_out/c5d/c5_d${d}_r$rep.err
done; done
