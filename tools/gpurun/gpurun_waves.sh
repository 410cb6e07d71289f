mkdir -p gpurun_out/waves
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -4 > gpurun_out/waves/tests.log
for i in 1 2; do
timeout 600 python bench.py --no-extra --no-predictor > gpurun_out/waves/bench_w$i.log 2> gpurun_out/waves/bench_w$i.err
HG_NO_WAVES=1 timeout 600 python bench.py --no-extra --no-predictor > gpurun_out/waves/bench_nw$i.log 2> gpurun_out/waves/bench_nw$i.err
done
timeout 300 python tools/prof_step.py c1 > gpurun_out/waves/prof_step.log 2>&1
