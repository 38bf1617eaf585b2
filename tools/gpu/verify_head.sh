# Round-end check of HEAD on a fresh box: GPU suite, smoke, the driver's default
# bench line (N=1, no flags) and the reference arm.
mkdir -p gpurun_out/verify
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/verify/gputests.log 2>&1; echo "rc=$?" >> gpurun_out/verify/gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/verify/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/verify/smoke.log
timeout 900 python bench.py > gpurun_out/verify/bench.json 2> gpurun_out/verify/bench.err; echo "rc=$?" >> gpurun_out/verify/bench.err
timeout 900 python bench.py --impl reference > gpurun_out/verify/bench_reference.json 2> gpurun_out/verify/bench_reference.err
