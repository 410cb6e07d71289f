# the final code: GPU suite (parity log), the -DHG_CHECKS build over the suite, smoke, bench line,
# 2-rank bench path on one GPU, reference arm, ncu launch list + --set full of the dominant kernels
mkdir -p gpurun_out/r2_final5
O=gpurun_out/r2_final5
export HG_PARITY_LOG=$PWD/$O/parity.log
timeout 1800 python -m pytest tests -m gpu -q -x -p no:cacheprovider > $O/tests.log 2>&1
echo rc=$? >> $O/tests.log
unset HG_PARITY_LOG
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
echo smoke_rc=$? >> $O/smoke.log
timeout 1500 python bench.py > $O/bench.log 2> $O/bench.err
echo bench_rc=$? >> $O/bench.err
HG_BENCH_SAME_GPU=1 timeout 600 python bench.py --gpus 2 --steps 20 --warmup 3 > $O/bench_g2_samegpu.log 2>&1
echo rc=$? >> $O/bench_g2_samegpu.log
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_ref.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"splitk|tc_attn|combine|append|barrier" \
    -c 400 --csv --log-file $O/launches_c3.csv \
    python bench.py --profile --no-extra --no-predictor --steps 20 --warmup 3 > $O/bench_under_ncu.log 2>&1
for c in p1 p2; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc_attn -c 1 -s 3 \
      -o $O/full_${c}_tc python tools/run_config.py $c --steps 5 > /dev/null 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:splitk -c 1 -s 3 \
    -o $O/full_c3_splitk python tools/run_config.py c3 --steps 5 > /dev/null 2>&1
export HG_SO_OVERRIDE=$PWD/paper_2501_14808_b200/var/libhygen_checks.so
python -c "import paper_2501_14808_b200 as hg; print('loaded', hg.SO_PATH)" > $O/checks.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider >> $O/checks.log 2>&1
echo rc=$? >> $O/checks.log
grep -c "HG_DCHECK failed" $O/checks.log >> $O/checks.log
