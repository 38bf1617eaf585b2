# PDL on/off A/B over every bench config (3 timed steps each)
mkdir -p gpurun_out/pdl
for cfg in 1 2 3 4 5; do
  for pdl in 0 1; do
    BS_PDL=$pdl timeout 900 python bench.py --config $cfg --steps 3 --warmup 3 --cpu-forward 0 \
      > gpurun_out/pdl/c${cfg}_pdl${pdl}.json 2> gpurun_out/pdl/c${cfg}_pdl${pdl}.err
  done
done
