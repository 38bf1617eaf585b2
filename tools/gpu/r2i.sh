mkdir -p gpurun_out/r2
timeout 900 python -m pytest tests/test_kernels_gpu.py -x -q -k "bf16 or cluster" > gpurun_out/r2/pytest_bf16.txt 2>&1; tail -n 25 gpurun_out/r2/pytest_bf16.txt
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r2/pytest_i.txt 2>&1; tail -n 5 gpurun_out/r2/pytest_i.txt
bash tools/gpu/r2h.sh
