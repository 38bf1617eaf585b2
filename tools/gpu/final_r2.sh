# Round-2 evidence: GPU tests, the reference-arm tables (bench.py's startup
# table per config), every bench config (+ bf16, the reference arm), the bench
# launch list, a full ncu capture of the top conv shapes.
mkdir -p gpurun_out/final/tables
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/final/gputests.log 2>&1; echo "rc=$?" >> gpurun_out/final/gputests.log
timeout 1500 python tools/bench_tables.py gpurun_out/final/tables > gpurun_out/final/tables.log 2>&1
cp gpurun_out/final/tables/*_table_b200.json profiles/r02/
for cfg in 2 1 3 4 5; do
  timeout 900 python bench.py --config $cfg > gpurun_out/final/bench_config$cfg.json 2> gpurun_out/final/bench_config$cfg.err
done
timeout 900 python bench.py --precision bf16 > gpurun_out/final/bench_config2_bf16.json 2> gpurun_out/final/bench_config2_bf16.err
timeout 900 python bench.py --impl reference > gpurun_out/final/bench_reference.json 2> gpurun_out/final/bench_reference.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/final/launches_bench.csv \
  python bench.py --steps 2 --warmup 3 --cpu-forward 0 > /dev/null 2>&1
for c in "90 56 64 192 3 1 1" "90 28 96 128 3 1 1" "90 224 4 64 7 2 3"; do
  n=$(echo $c | tr ' ' '_')
  timeout 300 ncu --set full --clock-control none -k regex:conv_tc -s 3 -c 1 -o gpurun_out/final/full_$n python tools/conv_case.py $c 5 > /dev/null 2>&1
done
