# GPU replay tests for configs 4/5 + bench lines for configs 1, 3, 4
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_executor_gpu.py -x -q -k "hetero3 or collab" > gpurun_out/cfg_tests.log 2>&1; tail -3 gpurun_out/cfg_tests.log
for c in 3 4 1; do timeout 900 python bench.py --config $c --steps 3 > gpurun_out/bench_c$c.json 2> gpurun_out/bench_c$c.err; echo "config $c rc=$?"; tail -c 300 gpurun_out/bench_c$c.json; echo; done
