# DRAM traffic per conv_tc launch over the config-2 workload population
# (profiles/ncu_conv_summary.json, bench.py roofline.traffic), and full ncu
# captures of the top conv shapes with the final kernel.
mkdir -p gpurun_out/traffic
timeout 900 ncu --profile-from-start off --clock-control none \
  --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv \
  --log-file gpurun_out/traffic/launches.csv python tools/traffic_replay.py gpurun_out/traffic/stats.json 600 \
  > gpurun_out/traffic/replay.log 2>&1; echo "rc=$?" >> gpurun_out/traffic/replay.log
python tools/traffic_summary.py gpurun_out/traffic/launches.csv gpurun_out/traffic/stats.json gpurun_out/traffic/ncu_conv_summary.json > gpurun_out/traffic/summary.log 2>&1
for c in "90 56 64 192 3 1 1" "90 28 96 128 3 1 1" "90 224 4 64 7 2 3"; do
  n=$(echo $c | tr ' ' '_')
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:conv_tc -s 3 -c 1 -o gpurun_out/traffic/full_$n python tools/conv_case.py $c 5 > /dev/null 2>&1
done
gzip -f gpurun_out/traffic/launches.csv
