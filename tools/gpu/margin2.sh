# A/B: planning margin on the latency table, config 2 (second sweep).
mkdir -p gpurun_out/margin2
for rep in 1 2; do for m in 1.06 1.10 1.15; do
  BENCH_TABLE_MARGIN=$m timeout 900 python bench.py --cpu-forward 0 > gpurun_out/margin2/c2_m${m}_r$rep.json 2> gpurun_out/margin2/c2_m${m}_r$rep.err
done; done
for m in 1.0 1.06; do
  BENCH_TABLE_MARGIN=$m timeout 900 python bench.py --config 5 > gpurun_out/margin2/c5_m${m}.json 2> gpurun_out/margin2/c5_m${m}.err
done
