# racecheck (shared-memory hazards) on a small selection: toy configs on both routes, the fused
# tcgen05 step (prologue and background append), a fuzz seed, the host step
mkdir -p gpurun_out/r2_race
T=tests/test_gpu_parity.py
SEL="$T::test_toy $T::test_fused_step_equals_append_then_attention[toy_a-0] $T::test_fused_step_equals_append_then_attention[toy_a-1] $T::test_fuzz[3] $T::test_e2e_host_step_matches_device_path[toy_a]"
timeout 2400 compute-sanitizer --tool racecheck --racecheck-report hazard --error-exitcode 9 --print-limit 20 \
    python -m pytest $SEL -q -x -p no:cacheprovider > gpurun_out/r2_race/racecheck.log 2>&1
echo "racecheck rc=$?" >> gpurun_out/r2_race/racecheck.log
