# Round-2 evidence of the final code: full GPU suite (whole-tensor parity log), smoke, the
# default bench line, the multi-rank bench path on one GPU, the reference arm, the ncu launch
# list of the bench command and of the sharded step, ncu --set full of the dominant kernels,
# the -DHG_CHECKS build over the whole GPU suite, the 8-rank bench path on one GPU
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
# compute-sanitizer is closed on this pool: the device-side checking build over the whole suite
export HG_SO_OVERRIDE=$PWD/paper_2501_14808_b200/var/libhygen_checks.so
python -c "import paper_2501_14808_b200 as hg; print('loaded', hg.SO_PATH)" > $O/checks.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider >> $O/checks.log 2>&1
echo rc=$? >> $O/checks.log
grep -c "HG_DCHECK failed" $O/checks.log >> $O/checks.log
unset HG_SO_OVERRIDE
HG_BENCH_SAME_GPU=1 timeout 1200 python bench.py --gpus 8 --steps 5 --warmup 3 > $O/bench_g8_samegpu.log 2>&1
echo rc=$? >> $O/bench_g8_samegpu.log
