mkdir -p gpurun_out/pdl35
for cfg in 3 5; do for p in 0 1; do
  BS_PDL=$p timeout 900 python bench.py --config $cfg --steps 3 --cpu-forward 0 > gpurun_out/pdl35/c${cfg}_pdl$p.json 2>/dev/null
done; done
