# Round-2 evidence of the final code: full GPU suite (whole-tensor parity log), smoke, the
# default bench line, the multi-rank bench path on one GPU, the reference arm, the ncu launch
# list of the bench command and of the sharded step, ncu --set full of the dominant kernels,
# compute-sanitizer memcheck / racecheck / synccheck on the paths this round changed
mkdir -p gpurun_out/r2_final
O=gpurun_out/r2_final
export HG_PARITY_LOG=$PWD/$O/parity.log
timeout 1800 python -m pytest tests -m gpu -q -x -p no:cacheprovider > $O/tests.log 2>&1
echo rc=$? >> $O/tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
echo smoke_rc=$? >> $O/smoke.log
timeout 1500 python bench.py > $O/bench.log 2> $O/bench.err
echo bench_rc=$? >> $O/bench.err
HG_BENCH_SAME_GPU=1 timeout 600 python bench.py --gpus 2 --steps 20 --warmup 3 > $O/bench_g2_samegpu.log 2>&1
echo rc=$? >> $O/bench_g2_samegpu.log
HG_BENCH_SAME_GPU=1 timeout 900 python bench.py --gpus 4 --steps 10 --warmup 3 > $O/bench_g4_samegpu.log 2>&1
echo rc=$? >> $O/bench_g4_samegpu.log
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_ref.log 2>&1
unset HG_PARITY_LOG
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"splitk|tc_attn|combine|append|barrier" \
    -c 400 --csv --log-file $O/launches_c3.csv \
    python bench.py --profile --no-extra --no-predictor --steps 20 --warmup 3 > $O/bench_under_ncu.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"splitk|tc_attn|combine|append|barrier" \
    --csv --log-file $O/launches_tp_c3g8.csv python tools/tp_launches.py c3 8 3 > $O/tp_launches.log 2>&1
for c in "c3" "c3@8" "c1"; do
  n=$(echo $c | tr '@' 'g')
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:splitk -c 1 -s 3 \
      -o $O/full_${n}_splitk python tools/run_config.py $c --steps 5 > /dev/null 2>&1
done
for c in p1 p2; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc_attn -c 1 -s 3 \
      -o $O/full_${c}_tc python tools/run_config.py $c --steps 5 > /dev/null 2>&1
done
T=tests/test_gpu_parity.py
P=tests/test_gpu_peer.py
SEL="$T::test_toy $T::test_fused_step_equals_append_then_attention $T::test_fuzz[0] $T::test_fuzz[3] $T::test_fuzz[7] $T::test_nested_fuzz[2] $T::test_plan_variants[0-tc_route] $T::test_plan_variants[1-hbm_route] $T::test_plan_variants[2-route3] $T::test_e2e_host_step_matches_device_path[toy_a] $T::test_e2e_host_step_pageable_output[toy_a] $T::test_prefill_key_split[c4_small_chunk] $P::test_window_world1 $P::test_window_world1_sharded_hbm_step_two_launches"
for tool in memcheck synccheck; do
  echo "== $tool" >> $O/san.log
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 \
      python -m pytest $SEL -q -x -p no:cacheprovider > $O/san_$tool.log 2>&1
  echo "$tool rc=$?" >> $O/san.log
  grep -E "ERROR SUMMARY|passed|failed" $O/san_$tool.log | tail -3 >> $O/san.log
done
RSEL="$T::test_toy $T::test_fused_step_equals_append_then_attention[toy_a-0] $T::test_fused_step_equals_append_then_attention[toy_a-1] $T::test_fuzz[3] $T::test_e2e_host_step_matches_device_path[toy_a] $P::test_window_world1_sharded_hbm_step_two_launches"
echo "== racecheck" >> $O/san.log
timeout 2400 compute-sanitizer --tool racecheck --racecheck-report hazard --error-exitcode 9 --print-limit 20 \
    python -m pytest $RSEL -q -x -p no:cacheprovider > $O/san_racecheck.log 2>&1
echo "racecheck rc=$?" >> $O/san.log
grep -E "RACECHECK SUMMARY|passed|failed" $O/san_racecheck.log | tail -3 >> $O/san.log
