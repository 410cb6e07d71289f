mkdir -p gpurun_out/e2e3
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "e2e" 2>&1 | tail -3 > gpurun_out/e2e3/tests.log
timeout 300 python tools/prof_e2e.py c1 > gpurun_out/e2e3/prof.log 2>&1
timeout 900 python bench.py --no-extra --no-predictor > gpurun_out/e2e3/bench.log 2> gpurun_out/e2e3/bench.err
