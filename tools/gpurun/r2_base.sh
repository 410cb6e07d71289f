mkdir -p gpurun_out/r2_base
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2_base/gpu.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -5 > gpurun_out/r2_base/tests.log
timeout 1200 python bench.py > gpurun_out/r2_base/bench.log 2> gpurun_out/r2_base/bench.err
echo bench=$? >> gpurun_out/r2_base/tests.log
