mkdir -p gpurun_out/slo2
timeout 900 python bench.py --no-extra > gpurun_out/slo2/bench.log 2> gpurun_out/slo2/bench.err
