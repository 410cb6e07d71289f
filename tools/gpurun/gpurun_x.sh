mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "fused or append or toy or fuzz1 or e2e" 2>&1 | tail -2 > gpurun_out/x.log
timeout 200 python tools/prof_step.py c1 > gpurun_out/prof_c1.log 2>&1
timeout 200 python tools/prof_step.py c3 > gpurun_out/prof_c3.log 2>&1
