# configs 3/4 accounting + GPU parity with calibrated weights
mkdir -p gpurun_out/r2
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r2/pytest_gpu.txt 2>&1; tail -5 gpurun_out/r2/pytest_gpu.txt
timeout 600 python tools/cfg_diag.py 4 1000 2000 3000 5000 8000 > gpurun_out/r2/diag4.txt 2>&1
timeout 600 python tools/cfg_diag.py 3 1000 2000 4000 8000 > gpurun_out/r2/diag3.txt 2>&1
tail -n 3 gpurun_out/r2/diag*.txt
