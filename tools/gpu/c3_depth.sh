mkdir -p gpurun_out/c3d
for rep in 1 2; do for d in 2 4; do
  BENCH_DEPTH=$d timeout 900 python bench.py --config 3 > gpurun_out/c3d/c3_d${d}_r$rep.json 2> gpurun_out/c3d/c3_d${d}_r$rep.err
done; done
