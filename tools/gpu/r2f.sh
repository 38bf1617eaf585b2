mkdir -p gpurun_out/r2
for b in 1 8; do
timeout 600 ncu --nvtx --nvtx-include "pass/" --cache-control none --clock-control none --metrics gpu__time_duration.sum --csv --log-file gpurun_out/r2/pass_goog_b$b.csv python tools/pass_launches.py googlenet $b > gpurun_out/r2/pass_goog_b$b.log 2>&1
done
ls -la gpurun_out/r2/pass_goog*
