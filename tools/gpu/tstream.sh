mkdir -p gpurun_out/ts
timeout 600 python -m pytest tests/test_executor_gpu.py -x -q > gpurun_out/ts/et.log 2>&1; echo "rc=$?" >> gpurun_out/ts/et.log
for r in 1 2; do for t in 0 1; do
  BS_TABLE_STREAM=$t timeout 900 python bench.py --steps 3 --cpu-forward 0 > gpurun_out/ts/c2_t${t}_$r.json 2>/dev/null
done; done
for t in 0 1; do BS_TABLE_STREAM=$t timeout 900 python bench.py --config 3 --steps 3 --cpu-forward 0 > gpurun_out/ts/c3_t${t}.json 2>/dev/null; done
