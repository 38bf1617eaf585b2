# Reference admission of HBM-resident images + skip of landed-copy waits:
# full GPU suite, then per-step excess and capacity ladder.
mkdir -p gpurun_out/zcadmit
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/zcadmit/gputests.log 2>&1; echo "rc=$?" >> gpurun_out/zcadmit/gputests.log
timeout 300 python tools/step_times.py 2 45000 > gpurun_out/zcadmit/steptimes_45000.txt 2>&1
timeout 900 python tools/table_capacity_ab.py 2 45000 48000 51000 54000 --modes=step > gpurun_out/zcadmit/cap.txt 2>&1
