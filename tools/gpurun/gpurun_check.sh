mkdir -p gpurun_out/check2
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3 > gpurun_out/check2/tests.log
