mkdir -p gpurun_out/c1g
for rep in 1 2; do for v in 0 1; do
  BS_FC_GEMV=$v timeout 900 python bench.py --config 1 > gpurun_out/c1g/c1_g${v}_r$rep.json 2> gpurun_out/c1g/c1_g${v}_r$rep.err
done; done
