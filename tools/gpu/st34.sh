mkdir -p gpurun_out/st34
BY_BATCH= timeout 600 python tools/step_times.py 3 7000 > gpurun_out/st34/c3_7000.txt 2>&1
timeout 600 python tools/step_times.py 4 13000 > gpurun_out/st34/c4_13000.txt 2>&1
