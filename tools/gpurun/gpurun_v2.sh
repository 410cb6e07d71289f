mkdir -p gpurun_out
timeout 400 python -m pytest tests/test_gpu_parity.py -q -x -k "toy or fuzz1 or p1 or p2 or peaked or nested_fuzz or head_dim_64 or gqa or max_context" 2>&1 | tail -2 > gpurun_out/v2.log
for c in p1 p2 c1_long; do timeout 120 python tools/run_config.py $c --time --steps 4 2>&1 | grep "^[pc]" | cut -c1-90 >> gpurun_out/v2.log; done
timeout 120 python tools/trace_tc.py p2 > gpurun_out/v2_trace.log 2>&1
