# Every bench config with the final code (+ bf16), for profiles/r02/head/.
mkdir -p gpurun_out/cfg
for cfg in 1 3 4 5; do
  timeout 900 python bench.py --config $cfg > gpurun_out/cfg/bench_config$cfg.json 2> gpurun_out/cfg/bench_config$cfg.err
done
timeout 900 python bench.py --precision bf16 > gpurun_out/cfg/bench_config2_bf16.json 2> gpurun_out/cfg/bench_config2_bf16.err
