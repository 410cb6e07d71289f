# tcgen05 V3 (quad-per-row softmax, 640 threads): a short parity probe first (bounded), then
# timing vs the default kernel, then the tcgen05-heavy parity selection
mkdir -p gpurun_out/r2_v3
export HG_TC_V3=1
timeout 180 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "test_toy and 1.0" > gpurun_out/r2_v3/probe.log 2>&1
echo rc=$? >> gpurun_out/r2_v3/probe.log
if grep -q "rc=0" gpurun_out/r2_v3/probe.log; then
  timeout 300 python tools/exp_tc.py p1 p2 > gpurun_out/r2_v3/exp.log 2>&1
  unset HG_TC_V3
  timeout 300 python tools/exp_tc.py p1 p2 >> gpurun_out/r2_v3/exp.log 2>&1
  export HG_TC_V3=1
  timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider --timeout 300 \
      -k "toy or fuzz or whole_tensor or peaked or prefill_key_split or plan_variants or gqa or head_dim or prefix_group or fused or e2e" > gpurun_out/r2_v3/tests.log 2>&1
  echo rc=$? >> gpurun_out/r2_v3/tests.log
  timeout 300 python tools/trace_tc.py p2 > gpurun_out/r2_v3/trace_p2.log 2>&1
fi
