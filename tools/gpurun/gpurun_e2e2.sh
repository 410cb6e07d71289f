mkdir -p gpurun_out/e2e
timeout 300 python tools/prof_step.py c1 > gpurun_out/e2e/prof_step.log 2>&1
timeout 900 python bench.py --no-extra > gpurun_out/e2e/bench.log 2> gpurun_out/e2e/bench.err
