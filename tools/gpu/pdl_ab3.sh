mkdir -p gpurun_out/pdl3
for cfg in 5 3 2; do
  for pdl in 0 1; do
    BS_PDL=$pdl timeout 900 python bench.py --config $cfg --steps 3 --warmup 3 --cpu-forward 0 \
      > gpurun_out/pdl3/c${cfg}_pdl${pdl}.json 2> gpurun_out/pdl3/c${cfg}_pdl${pdl}.err
  done
done
