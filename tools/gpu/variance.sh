# Run-to-run spread of the default bench line (config 2) at HEAD.
mkdir -p gpurun_out/var
for rep in 1 2 3; do
  timeout 900 python bench.py > gpurun_out/var/c2_r$rep.json 2> gpurun_out/var/c2_r$rep.err
done
