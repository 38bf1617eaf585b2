# Full GPU parity + conv shape timings + per-network layer sums at b=90.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/par_full.txt 2>&1; tail -1 gpurun_out/par_full.txt
DEBUGS="0" bash tools/gpu/epiab.sh
