# e2e host step, zero-copy result (final): host-step parity, wall time A/B on C3 / c1 / c2
mkdir -p gpurun_out/r2_zc2
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider --timeout 600 \
    -k "e2e or toy or error" > gpurun_out/r2_zc2/tests.log 2>&1
echo rc=$? >> gpurun_out/r2_zc2/tests.log
for c in c3 c1 c2; do
  HG_E2E_TRACE=1 timeout 300 python tools/prof_e2e.py $c > gpurun_out/r2_zc2/prof_$c.log 2> gpurun_out/r2_zc2/prof_$c.err
  HG_E2E_NO_ZC=1 timeout 300 python tools/prof_e2e.py $c > gpurun_out/r2_zc2/prof_${c}_nozc.log 2>&1
done
