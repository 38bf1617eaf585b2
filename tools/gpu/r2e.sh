mkdir -p gpurun_out/r2
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r2/pytest_tune.txt 2>&1; tail -n 5 gpurun_out/r2/pytest_tune.txt
TUNE_LOG=gpurun_out/r2/tunelog timeout 900 python tools/tuned_span.py small_cnn:1,10 googlenet:1,4,8,16,32,90 resnet50:1,8,32,90 mobilenet_v2:1,8,32 > gpurun_out/r2/tuned_span.txt 2>&1
cat gpurun_out/r2/tuned_span.txt
