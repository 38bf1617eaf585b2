# Stem attribution (7x7/2, Cin 4 -> 64 at 224x224, b=90) + launch list of GoogLeNet layer 1.
mkdir -p gpurun_out
for d in 0 4 32; do
  BS_CONV_DEBUG=$d timeout 120 python -c "
from tools.conv_bench import bench
print('debug=$d stem 7x7/2 224 4->64: %.1f us' % bench(90, 224, 4, 64, 7, 3, reps=10, stride=2))"
done
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/ll_g1.csv python tools/run_layers.py googlenet --batch 90 --from 1 --to 3 --reps 1 > /dev/null 2>&1
python - <<PY
import csv
rows=[r for r in csv.reader(open("gpurun_out/ll_g1.csv")) if len(r)>10]
h=rows[0]; ik=h.index("Kernel Name"); im=h.index("Metric Name"); iv=h.index("Metric Value"); iid=h.index("ID")
d={}
for r in rows[1:]: d.setdefault(r[iid],[r[ik][:50],{}])[1][r[im]]=r[iv]
for k,(n,m) in d.items(): print(k,n,m.get("gpu__time_duration.sum"),m.get("dram__bytes_read.sum"),m.get("dram__bytes_write.sum"))
PY
