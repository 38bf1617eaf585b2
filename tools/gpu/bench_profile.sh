# round evidence: bench line, launch list of the bench command (first 3000 launches), one full ncu capture of conv_tc
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 1 --warmup 3 > gpurun_out/bench_under_ncu.log 2>&1; echo "ncu list rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:conv_tc -s 40 -c 3 -o gpurun_out/prof_conv python tools/run_layers.py googlenet --batch 32 --reps 1 > gpurun_out/prof_conv.log 2>&1; echo "ncu full b32 rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:conv_tc -s 12 -c 3 -o gpurun_out/prof_conv90 python tools/run_layers.py googlenet --batch 90 --from 5 --to 8 --reps 1 > gpurun_out/prof_conv90.log 2>&1; echo "ncu full b90 rc=$?"
