mkdir -p gpurun_out/c4ab
DEPTHS=4 timeout 1500 python tools/table_capacity_ab.py 4 11000 15000 --modes=pass,step > gpurun_out/c4ab/c4_rev.txt 2>&1
DEPTHS=4 timeout 1500 python tools/table_capacity_ab.py 3 8000 10000 --modes=pass,step > gpurun_out/c4ab/c3.txt 2>&1
