mkdir -p gpurun_out/stem
python -m pytest tests/test_kernels_gpu.py -x -q > gpurun_out/stem/kt.log 2>&1
for rw in 0 1; do
  echo "rowwin=$rw stem b=90: $(BS_CONV_ROWWIN=$rw python tools/conv_case.py 90 224 4 64 7 2 3 20)"
  echo "rowwin=$rw stem b=8: $(BS_CONV_ROWWIN=$rw python tools/conv_case.py 8 224 4 64 7 2 3 20)"
  echo "rowwin=$rw stem b=1: $(BS_CONV_ROWWIN=$rw python tools/conv_case.py 1 224 4 64 7 2 3 20)"
done > gpurun_out/stem/times.txt 2>&1
