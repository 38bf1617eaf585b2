mkdir -p gpurun_out/r2
timeout 900 python bench.py --config 2 --cpu-forward 0 --deadline-ms 3.559 > gpurun_out/r2/bench3_c2_d3559.json 2> gpurun_out/r2/bench3_c2.err
timeout 900 python bench.py --config 2 --cpu-forward 0 --deadline-ms 3.559 --precision bf16 > gpurun_out/r2/bench3_c2_bf16.json 2> gpurun_out/r2/bench3_c2_bf16.err
for f in gpurun_out/r2/bench3_*.json; do python -c "
import json,sys
d=json.load(open('$f'))
print('$f', d['value'], d['on_time_ratio'], d['config']['deadline_ms'], d['config']['t1_ms'], d['config']['t_max_batch_ms'], d['e2e']['value'], d['roofline']['frac'], d['capacity_search'])
"; done
