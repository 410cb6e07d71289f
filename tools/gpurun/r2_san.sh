# compute-sanitizer over a subset of the parity tests (toy, fuzz, nested fuzz, both routes,
# the fused tcgen05 append, the host step) -- memcheck, racecheck, synccheck
mkdir -p gpurun_out/r2_san
SEL="test_toy or test_fuzz and not nested or test_plan_variants or test_fused_step_equals or test_e2e_host_step_matches_device_path and toy"
for tool in memcheck racecheck synccheck; do
  echo "== $tool" >> gpurun_out/r2_san/san.log
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 \
      python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "$SEL" >> gpurun_out/r2_san/san_$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/r2_san/san.log
  grep -E "ERROR SUMMARY|RACECHECK SUMMARY|passed|failed" gpurun_out/r2_san/san_$tool.log | tail -3 >> gpurun_out/r2_san/san.log
done
