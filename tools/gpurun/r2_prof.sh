# ncu launch list of the bench command (cold-cache, serialised per-launch times: compare
# shares, not absolutes) and --set full captures of the dominant kernels
mkdir -p gpurun_out/r2_prof
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"splitk|tc_attn|combine|append|barrier" \
    -c 400 --csv --log-file gpurun_out/r2_prof/launches_c3.csv \
    python bench.py --profile --no-extra --no-predictor --steps 20 --warmup 3 > gpurun_out/r2_prof/bench_under_ncu.log 2>&1
for c in "c3" "c3@8" "c1"; do
  n=$(echo $c | tr '@' 'g')
  ncu --set full --clock-control none --import-source on -k regex:splitk -c 1 -s 3 \
      -o gpurun_out/r2_prof/full_${n}_splitk python tools/run_config.py $c --steps 5 > /dev/null 2>&1
done
for c in p1 p2; do
  ncu --set full --clock-control none --import-source on -k regex:tc_attn -c 1 -s 3 \
      -o gpurun_out/r2_prof/full_${c}_tc python tools/run_config.py $c --steps 5 > /dev/null 2>&1
done
for c in c3@8 c3@4 c3 c1@8 c1; do timeout 300 python tools/trace_sk.py $c; done > gpurun_out/r2_prof/trace_sk.log 2>&1
