# Latency-table timing mode (step vs pass) -> served capacity, config 2; and
# the step-stamped per-step excess with the step table.
mkdir -p gpurun_out/tcap
timeout 900 python tools/table_capacity_ab.py 2 42000 45000 48000 51000 54000 > gpurun_out/tcap/c2.txt 2>&1
timeout 300 python tools/step_times.py 2 45000 > gpurun_out/tcap/steptimes_c2_45000.txt 2>&1
