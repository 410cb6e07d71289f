mkdir -p gpurun_out/slo
timeout 900 python bench.py --no-extra > gpurun_out/slo/bench.log 2> gpurun_out/slo/bench.err
