set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -30 > gpurun_out/r2a_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2a_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/r2a_bench.log 2>&1
timeout 600 python bench.py --impl reference > gpurun_out/r2a_ref.log 2>&1
tail -3 gpurun_out/r2a_*.log
