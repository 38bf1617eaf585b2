mkdir -p gpurun_out/zc
BS_ADMIT_ZC=1 timeout 600 python -m pytest tests/test_executor_gpu.py -x -q -k "h2d or live" > gpurun_out/zc/t.log 2>&1; echo "rc=$?" >> gpurun_out/zc/t.log
for z in 0 1; do BS_ADMIT_ZC=$z timeout 900 python bench.py --steps 3 --cpu-forward 0 > gpurun_out/zc/c2_zc$z.json 2>/dev/null; done
