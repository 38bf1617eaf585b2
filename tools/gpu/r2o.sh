mkdir -p gpurun_out/r2
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r2/pytest_o.txt 2>&1; tail -n 5 gpurun_out/r2/pytest_o.txt
timeout 600 python tools/tuned_span.py googlenet:1,8,90 resnet50:1,90 > gpurun_out/r2/tuned_span3.txt 2>&1; cat gpurun_out/r2/tuned_span3.txt
timeout 300 python tools/live_scale.py 3.559 2>&1 | head -1
