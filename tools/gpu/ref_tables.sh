# Refresh the reference arm's B200 tables with the final code, then the reference arm.
mkdir -p gpurun_out/rt/tables
timeout 1500 python tools/bench_tables.py gpurun_out/rt/tables > gpurun_out/rt/tables.log 2>&1
cp gpurun_out/rt/tables/*_table_b200.json profiles/r02/
timeout 900 python bench.py --impl reference > gpurun_out/rt/bench_reference_arm.json 2> gpurun_out/rt/bench_reference_arm.err
for c in 3 4; do timeout 900 python bench.py --impl reference --config $c > gpurun_out/rt/bench_reference_arm_c$c.json 2> gpurun_out/rt/bench_reference_arm_c$c.err; done
