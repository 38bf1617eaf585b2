# Config 3: planning margin and steps in flight (sparse sampling protocol).
mkdir -p gpurun_out/c3t
for m in 1.0 1.1 1.2; do
  BENCH_TABLE_MARGIN=$m timeout 900 python bench.py --config 3 > gpurun_out/c3t/c3_m${m}.json 2> gpurun_out/c3t/c3_m${m}.err
done
BENCH_DEPTH=3 timeout 900 python bench.py --config 3 > gpurun_out/c3t/c3_d3.json 2> gpurun_out/c3t/c3_d3.err
BENCH_DEPTH=2 timeout 900 python bench.py --config 3 > gpurun_out/c3t/c3_d2.json 2> gpurun_out/c3t/c3_d2.err
