# Per-step extras (table-write kernel, step mark, event) on one-layer-step passes.
mkdir -p gpurun_out/step_chain
for s in googlenet resnet50; do timeout 600 python tools/step_chain.py $s 1 10 40 90; done > gpurun_out/step_chain/times.txt 2>&1
