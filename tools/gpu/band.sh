mkdir -p gpurun_out/band
timeout 300 python -m pytest tests/test_kernels_gpu.py -x -q -k "maxpool" > gpurun_out/band/kt.log 2>&1; echo "rc=$?" >> gpurun_out/band/kt.log
for b in 0 1; do for a in "googlenet 90" "googlenet 8" "googlenet 1"; do BS_POOL_BAND=$b timeout 300 python tools/b1_anatomy.py $a | sed "s/^/band=$b /"; done; done > gpurun_out/band/times.txt 2>&1
BS_POOL_BAND=1 bash tools/gpu/pass_ncu.sh googlenet 90
