# Live-loop per-step device time vs table prediction (config 2 near capacity),
# stamped by the table-write kernels; per-step extras offline (step_chain).
mkdir -p gpurun_out/steptimes
timeout 600 python -m pytest tests/test_executor_gpu.py -x -q > gpurun_out/steptimes/exec_tests.log 2>&1; echo "rc=$?" >> gpurun_out/steptimes/exec_tests.log
for r in 40000 45000; do
  echo "== rate $r"
  timeout 300 python tools/step_times.py 2 $r gpurun_out/steptimes/c2_$r.json
done > gpurun_out/steptimes/summary.txt 2>&1
timeout 600 python tools/step_chain.py googlenet 1 10 40 90 > gpurun_out/steptimes/chain.txt 2>&1
