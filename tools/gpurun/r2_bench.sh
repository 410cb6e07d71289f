# the default bench line (+ smoke) of the final code
mkdir -p gpurun_out/r2_bench
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_bench/smoke.log 2>&1
echo smoke_rc=$? >> gpurun_out/r2_bench/smoke.log
timeout 1500 python bench.py > gpurun_out/r2_bench/bench.log 2> gpurun_out/r2_bench/bench.err
echo bench_rc=$? >> gpurun_out/r2_bench/bench.err
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider --timeout 600 -k "e2e or toy or plan_variants" > gpurun_out/r2_bench/tests.log 2>&1
echo rc=$? >> gpurun_out/r2_bench/tests.log
