# A/B: batched admission of GoogLeNet's 150 KB images (per-image DMA from the
# pinned pool, one expansion launch + ready event per loop iteration) vs one
# copy + expansion + event per request; config 2 e2e.
mkdir -p gpurun_out/bl
BS_BATCH_ADMIT_LARGE=1 timeout 600 python -m pytest tests/test_executor_gpu.py -m gpu -x -q -k "h2d" > gpurun_out/bl/tests.log 2>&1; echo "rc=$?" >> gpurun_out/bl/tests.log
for rep in 1 2; do for v in 0 1; do
  BS_BATCH_ADMIT_LARGE=$v timeout 900 python bench.py --cpu-forward 0 > gpurun_out/bl/c2_l${v}_r$rep.json 2> gpurun_out/bl/c2_l${v}_r$rep.err
done; done
