mkdir -p gpurun_out/check
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3 > gpurun_out/check/tests.log
