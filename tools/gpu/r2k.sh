mkdir -p gpurun_out/r2
timeout 900 python -m pytest tests/test_executor_gpu.py -q -s -k "bf16" > gpurun_out/r2/pytest_bf16_e2e.txt 2>&1; tail -n 12 gpurun_out/r2/pytest_bf16_e2e.txt
