# A/B: planning margin on the latency table (config 2, and config 4).
mkdir -p gpurun_out/margin
for rep in 1 2; do for m in 1.0 1.03 1.06; do
  BENCH_TABLE_MARGIN=$m timeout 900 python bench.py --cpu-forward 0 > gpurun_out/margin/c2_m${m}_r$rep.json 2> gpurun_out/margin/c2_m${m}_r$rep.err
done; done
for m in 1.0 1.04; do
  BENCH_TABLE_MARGIN=$m timeout 900 python bench.py --config 4 > gpurun_out/margin/c4_m${m}.json 2> gpurun_out/margin/c4_m${m}.err
done
