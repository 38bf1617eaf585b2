mkdir -p gpurun_out
for d in 0 1 2 4 7; do echo "== BS_CONV_DEBUG=$d"; BS_CONV_DEBUG=$d timeout 120 python tools/conv_bench.py 2>&1 | grep "b=90" ; done
