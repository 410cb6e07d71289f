mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_rope.py -q -x 2>&1 | tail -15 > gpurun_out/r2_rope.log
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3 > gpurun_out/r2_tests.log
timeout 200 python tools/prof_step.py c1 > gpurun_out/prof_c1.log 2>&1
