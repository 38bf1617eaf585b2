mkdir -p gpurun_out/depth3
for d in 4 6 8; do echo "== depth $d"; DEPTH=$d timeout 600 python tools/table_capacity_ab.py 2 54000 57000 60000 --modes=step; done > gpurun_out/depth3/c2.txt 2>&1
