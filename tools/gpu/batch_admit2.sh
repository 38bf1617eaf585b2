mkdir -p gpurun_out/badm2
timeout 900 python bench.py --config 1 > gpurun_out/badm2/bench_config1.json 2> gpurun_out/badm2/bench_config1.err
timeout 900 python bench.py > gpurun_out/badm2/bench_config2.json 2> gpurun_out/badm2/bench_config2.err
