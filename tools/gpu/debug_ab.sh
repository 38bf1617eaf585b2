for d in 0 8 16 24 31; do echo "== BS_CONV_DEBUG=$d"; BS_CONV_DEBUG=$d timeout 120 python tools/conv_bench.py 2>&1 | grep "b=90" ; done
