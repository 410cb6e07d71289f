# e2e host step: zero-copy result + late wave on the HBM route: parity, then wall time A/B
mkdir -p gpurun_out/r2_late
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider --timeout 600 \
    -k "e2e or toy or error" > gpurun_out/r2_late/tests.log 2>&1
echo rc=$? >> gpurun_out/r2_late/tests.log
for c in c3 c1 c2 p1; do
  HG_E2E_TRACE=1 timeout 300 python tools/prof_e2e.py $c > gpurun_out/r2_late/prof_$c.log 2> gpurun_out/r2_late/prof_$c.err
  HG_E2E_NO_LATE=1 timeout 300 python tools/prof_e2e.py $c > gpurun_out/r2_late/prof_${c}_nolate.log 2>&1
done
