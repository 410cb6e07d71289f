mkdir -p gpurun_out; rm -f gpurun_out/k80.log
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "toy or fuzz1 or p1 or p2 or peaked or nested_fuzz or head_dim_64 or gqa or max_context" 2>&1 | tail -3 > gpurun_out/k80.log
for c in p1 p2 c1_long c1; do timeout 120 python tools/run_config.py $c --time --steps 4 2>&1 | grep "^[pc]" | cut -c1-90 >> gpurun_out/k80.log; done
timeout 120 python tools/trace_tc.py p2 > gpurun_out/k80_trace.log 2>&1
