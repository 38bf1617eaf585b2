mkdir -p gpurun_out/e2e
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/e2e/gputest.log 2>&1; echo "rc=$?" >> gpurun_out/e2e/gputest.log
for r in 1 2; do timeout 900 python bench.py --steps 3 --cpu-forward 0 > gpurun_out/e2e/c2_$r.json 2>/dev/null; done
