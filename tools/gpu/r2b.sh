# round 2: measured tables for the reference arm / parity fixtures + small-batch diagnostics
mkdir -p gpurun_out/r2 profiles/r02
timeout 900 python bench.py --config 2 --steps 3 --warmup 3 --cpu-forward 0 --dump-table profiles/r02/googlenet_table_b200.json > gpurun_out/r2/bench_c2.json 2> gpurun_out/r2/bench_c2.err
timeout 900 python bench.py --config 3 --steps 3 --warmup 3 --cpu-forward 0 --dump-table profiles/r02/resnet50_pair_table_b200.json > gpurun_out/r2/bench_c3.json 2> gpurun_out/r2/bench_c3.err
timeout 900 python bench.py --config 4 --steps 3 --warmup 3 --cpu-forward 0 --dump-table profiles/r02/hetero3_table_b200.json > gpurun_out/r2/bench_c4.json 2> gpurun_out/r2/bench_c4.err
timeout 600 python bench.py --config 1 --steps 3 --warmup 3 --cpu-forward 0 --dump-table profiles/r02/small_cnn_table_b200.json > gpurun_out/r2/bench_c1.json 2> gpurun_out/r2/bench_c1.err
cp profiles/r02/*.json gpurun_out/r2/
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2/ll_goog_b1.csv python tools/run_layers.py googlenet --batch 1 --reps 1 > /dev/null 2>&1
timeout 300 python tools/span_bench.py small_cnn:1,10 googlenet:1,8,32,90 resnet50:1,8 mobilenet_v2:1,8 > gpurun_out/r2/span.txt 2>&1
timeout 600 python tools/cfg_diag.py 3 1000 2000 4000 8000 > gpurun_out/r2/diag3.txt 2>&1
timeout 600 python tools/cfg_diag.py 4 1000 2000 3000 5000 8000 > gpurun_out/r2/diag4.txt 2>&1
tail -3 gpurun_out/r2/*.txt
