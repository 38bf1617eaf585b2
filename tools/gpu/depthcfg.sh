mkdir -p gpurun_out/depthcfg
DEPTHS=3,4 timeout 600 python tools/table_capacity_ab.py 1 80000 95000 --modes=step > gpurun_out/depthcfg/c1.txt 2>&1
DEPTHS=3,4 timeout 900 python tools/table_capacity_ab.py 3 7000 8500 --modes=step > gpurun_out/depthcfg/c3.txt 2>&1
DEPTHS=3,4 timeout 900 python tools/table_capacity_ab.py 4 13000 15000 --modes=step > gpurun_out/depthcfg/c4.txt 2>&1
