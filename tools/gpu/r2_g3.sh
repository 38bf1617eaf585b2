mkdir -p gpurun_out/r2
python tools/layer_err.py googlenet tf32x2 1 > gpurun_out/r2/lerr_goog.txt 2>&1; tail -3 gpurun_out/r2/lerr_goog.txt
python tools/layer_err.py resnet50 tf32x2 1 > gpurun_out/r2/lerr_r50.txt 2>&1; tail -3 gpurun_out/r2/lerr_r50.txt
timeout 300 python tools/span_bench.py small_cnn:1,10 googlenet:1,8,32,90 resnet50:1,8 mobilenet_v2:1,8 > gpurun_out/r2/span.txt 2>&1; cat gpurun_out/r2/span.txt
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/r2/pytest_gpu.txt 2>&1; tail -8 gpurun_out/r2/pytest_gpu.txt
