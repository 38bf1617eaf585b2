# Config-3 GPU replay test (every served request vs the oracle) and a
# functional N = 2 bench run (two ranks on GPU 0 over gloo: checks the sharded
# launch path, rank-consistent rates and rank-0 output; its timings mean nothing).
mkdir -p gpurun_out/c3n2
timeout 900 python -m pytest tests/test_executor_gpu.py -m gpu -x -q -k "config3 or config4 or riders" > gpurun_out/c3n2/tests.log 2>&1; echo "rc=$?" >> gpurun_out/c3n2/tests.log
BENCH_ONE_DEVICE=1 BENCH_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 1 --warmup 3 --requests 600 --warm-requests 600 --slots 1024 \
  > gpurun_out/c3n2/bench_n2.json 2> gpurun_out/c3n2/bench_n2.err; echo "rc=$?" >> gpurun_out/c3n2/bench_n2.err
