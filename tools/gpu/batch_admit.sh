# Batched H2D admission of small images: live-serving parity tests and the
# config-1 bench line (e2e), then config 2 (large images keep per-request DMA).
mkdir -p gpurun_out/badm
timeout 900 python -m pytest tests/test_executor_gpu.py -m gpu -x -q -k "live_serve" > gpurun_out/badm/tests.log 2>&1; echo "rc=$?" >> gpurun_out/badm/tests.log
timeout 900 python bench.py --config 1 > gpurun_out/badm/bench_config1.json 2> gpurun_out/badm/bench_config1.err
