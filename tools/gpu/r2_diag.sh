# round 2 first diagnostic: small-batch layer times + configs 3/4 accounting
mkdir -p gpurun_out/r2
for b in 1 10; do timeout 200 python tools/run_layers.py small_cnn --batch $b --reps 50 > gpurun_out/r2/small_b$b.txt 2>&1; done
for b in 1 8; do timeout 200 python tools/run_layers.py googlenet --batch $b --reps 20 > gpurun_out/r2/goog_b$b.txt 2>&1; done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2/ll_goog_b1.csv python tools/run_layers.py googlenet --batch 1 --reps 1 > /dev/null 2>&1
timeout 600 python tools/cfg_diag.py 4 1000 2000 3000 5000 8000 > gpurun_out/r2/diag4.txt 2>&1
timeout 600 python tools/cfg_diag.py 3 1000 2000 4000 8000 > gpurun_out/r2/diag3.txt 2>&1
tail -3 gpurun_out/r2/*.txt
