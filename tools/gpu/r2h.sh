mkdir -p gpurun_out/r2
timeout 900 python bench.py --config 2 --cpu-forward 0 > gpurun_out/r2/bench2_c2.json 2> gpurun_out/r2/bench2_c2.err
timeout 900 python bench.py --config 2 --cpu-forward 0 --table-flush-l2 1 > gpurun_out/r2/bench2_c2_cold.json 2> gpurun_out/r2/bench2_c2_cold.err
timeout 900 python bench.py --config 4 --steps 3 --cpu-forward 0 > gpurun_out/r2/bench2_c4.json 2> gpurun_out/r2/bench2_c4.err
timeout 900 python bench.py --config 3 --steps 3 --cpu-forward 0 > gpurun_out/r2/bench2_c3.json 2> gpurun_out/r2/bench2_c3.err
for f in gpurun_out/r2/bench2_*.json; do python -c "
import json,sys
d=json.load(open('$f'))
print('$f', d['value'], d['on_time_ratio'], d['config']['deadline_ms'], d['config']['t1_ms'], d['config']['t_max_batch_ms'], d['e2e']['value'], d['roofline']['frac'], d['capacity_search'])
"; done
