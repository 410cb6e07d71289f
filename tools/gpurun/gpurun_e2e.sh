mkdir -p gpurun_out/e2e
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "e2e" -s 2>&1 | tail -15 > gpurun_out/e2e/tests.log
timeout 900 python bench.py --no-extra > gpurun_out/e2e/bench.log 2> gpurun_out/e2e/bench.err
echo bench=$? >> gpurun_out/e2e/tests.log
