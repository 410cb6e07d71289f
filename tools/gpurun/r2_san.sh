# compute-sanitizer over a subset of the parity tests (toy, a few fuzz seeds incl. nested,
# both routes, the fused tcgen05 append, the host step) -- memcheck, racecheck, synccheck
mkdir -p gpurun_out/r2_san
T=tests/test_gpu_parity.py
SEL="$T::test_toy $T::test_fused_step_equals_append_then_attention $T::test_fuzz[0] $T::test_fuzz[3] $T::test_fuzz[7] $T::test_nested_fuzz[2] $T::test_plan_variants[0-tc_route] $T::test_plan_variants[1-hbm_route] $T::test_e2e_host_step_matches_device_path[toy_a] $T::test_prefill_key_split[c4_small_chunk]"
for tool in memcheck racecheck synccheck; do
  echo "== $tool" >> gpurun_out/r2_san/san.log
  timeout 1200 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 \
      python -m pytest $SEL -q -x -p no:cacheprovider > gpurun_out/r2_san/san_$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/r2_san/san.log
  grep -E "ERROR SUMMARY|RACECHECK SUMMARY|passed|failed" gpurun_out/r2_san/san_$tool.log | tail -3 >> gpurun_out/r2_san/san.log
done
