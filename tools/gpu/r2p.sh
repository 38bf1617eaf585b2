mkdir -p gpurun_out/r2
for pdl in 0 1; do
BS_PDL=$pdl timeout 600 python bench.py --config 2 --cpu-forward 0 --deadline-ms 3.559 > gpurun_out/r2/pdl${pdl}_c2.json 2>/dev/null
BS_PDL=$pdl timeout 600 python bench.py --config 3 --steps 3 --cpu-forward 0 > gpurun_out/r2/pdl${pdl}_c3.json 2>/dev/null
BS_PDL=$pdl timeout 600 python bench.py --config 4 --steps 3 --cpu-forward 0 > gpurun_out/r2/pdl${pdl}_c4.json 2>/dev/null
done
for f in gpurun_out/r2/pdl*.json; do python -c "
import json
d=json.load(open('$f'))
print('$f', d['value'], d['on_time_ratio'], d['config']['deadline_ms'], d['config']['t1_ms'], d['config']['t_max_batch_ms'], d['e2e']['value'], [(round(r),x) for r,x in d['capacity_search']])
"; done
