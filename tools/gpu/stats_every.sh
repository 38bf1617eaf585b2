# A/B: conv-launch event sampling density inside the timed region (config 2).
mkdir -p gpurun_out/sev
for rep in 1 2; do for e in 4 32 1000000000; do
  timeout 900 python bench.py --cpu-forward 0 --stats-every $e > gpurun_out/sev/c2_e${e}_r$rep.json 2> gpurun_out/sev/c2_e${e}_r$rep.err
done; done
