# the pipelined host step (plan the next step while the GPU runs, async call): parity of the
# host-step paths, then the bench line (its e2e now also reports the plan-ahead loop)
mkdir -p gpurun_out/r2_ahead
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider --timeout 600 \
    -k "e2e or toy or error" > gpurun_out/r2_ahead/tests.log 2>&1
echo rc=$? >> gpurun_out/r2_ahead/tests.log
timeout 1500 python bench.py > gpurun_out/r2_ahead/bench.log 2> gpurun_out/r2_ahead/bench.err
echo bench_rc=$? >> gpurun_out/r2_ahead/bench.err
