# Tables with the serving-step timing (for the reference arm), then config 2
# (both arms) on them.
mkdir -p gpurun_out/r2b/tables
timeout 1200 python tools/bench_tables.py gpurun_out/r2b/tables > gpurun_out/r2b/tables.log 2>&1
cp gpurun_out/r2b/tables/*_table_b200.json profiles/r02/
timeout 900 python bench.py > gpurun_out/r2b/bench_config2.json 2> gpurun_out/r2b/bench_config2.err
timeout 900 python bench.py --impl reference > gpurun_out/r2b/bench_reference.json 2> gpurun_out/r2b/bench_reference.err
