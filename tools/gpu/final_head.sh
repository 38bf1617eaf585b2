# Final evidence with the final bench protocol: every config (+ bf16) and the reference arm.
mkdir -p gpurun_out/fin
timeout 900 python bench.py > gpurun_out/fin/bench_config2.json 2> gpurun_out/fin/bench_config2.err
for cfg in 1 3 4 5; do
  timeout 900 python bench.py --config $cfg > gpurun_out/fin/bench_config$cfg.json 2> gpurun_out/fin/bench_config$cfg.err
done
timeout 900 python bench.py --precision bf16 > gpurun_out/fin/bench_config2_bf16.json 2> gpurun_out/fin/bench_config2_bf16.err
timeout 900 python bench.py --impl reference > gpurun_out/fin/bench_reference_arm.json 2> gpurun_out/fin/bench_reference_arm.err
