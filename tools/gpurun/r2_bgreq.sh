# background append by request (need order, per-request counters): p1 / p2 fused steps, parity
mkdir -p gpurun_out/r2_bgreq
timeout 300 python tools/exp_tc.py p1 p2 > gpurun_out/r2_bgreq/exp.log 2>&1
HG_NO_BG_APPEND=1 timeout 300 python tools/exp_tc.py p1 p2 >> gpurun_out/r2_bgreq/exp.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_rope.py -q -x -p no:cacheprovider --timeout 600 \
    -k "fused or whole_tensor or peaked or toy or e2e or prefill_key_split or fuzz or gqa or head_dim or prefix_group or c4" > gpurun_out/r2_bgreq/tests.log 2>&1
echo rc=$? >> gpurun_out/r2_bgreq/tests.log
