# Config 2 at a ladder of offered rates: live loop accounting (predicted vs
# device time, host time, step sizes) with and without per-launch stats.
mkdir -p gpurun_out/diag2
STATS=0 DEPTH=3 DEADLINE_MS=3.559 timeout 600 python tools/cfg_diag.py 2 30000 40000 45000 50000 > gpurun_out/diag2/stats0.txt 2>&1
STATS=1 DEPTH=3 DEADLINE_MS=3.559 timeout 600 python tools/cfg_diag.py 2 40000 50000 > gpurun_out/diag2/stats1.txt 2>&1
