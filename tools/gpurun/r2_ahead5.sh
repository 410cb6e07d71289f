# host step: descriptors on the input copy stream (behind wave 0, ahead of wave 1); plan-ahead A/B
mkdir -p gpurun_out/r2_ahead5
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider --timeout 600 \
    -k "e2e or toy or error" > gpurun_out/r2_ahead5/tests.log 2>&1
echo rc=$? >> gpurun_out/r2_ahead5/tests.log
timeout 400 python tools/e2e_ahead.py c3 > gpurun_out/r2_ahead5/c3.log 2>&1
timeout 400 python tools/e2e_ahead.py c1 > gpurun_out/r2_ahead5/c1.log 2>&1
