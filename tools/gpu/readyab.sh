mkdir -p gpurun_out/ready
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/ready/gputest.log 2>&1; echo "rc=$?" >> gpurun_out/ready/gputest.log
for r in 1 2; do timeout 900 python bench.py --steps 3 --cpu-forward 0 > gpurun_out/ready/c2_$r.json 2>/dev/null; done
timeout 900 python bench.py --config 5 --steps 3 --cpu-forward 0 > gpurun_out/ready/c5.json 2>/dev/null
timeout 900 python bench.py --config 3 --steps 3 --cpu-forward 0 > gpurun_out/ready/c3.json 2>/dev/null
