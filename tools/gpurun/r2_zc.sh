# e2e host step with the zero-copy result (split-K / combine rows stored into the pinned
# out_host by the kernels): parity of the host-step paths, then C3 / c1 / c2 wall time A/B
mkdir -p gpurun_out/r2_zc
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider --timeout 600 \
    -k "e2e or toy or error" > gpurun_out/r2_zc/tests.log 2>&1
echo rc=$? >> gpurun_out/r2_zc/tests.log
for c in c3 c1 c2; do
  HG_E2E_TRACE=1 timeout 300 python tools/prof_e2e.py $c > gpurun_out/r2_zc/prof_$c.log 2> gpurun_out/r2_zc/prof_$c.err
  HG_E2E_NO_ZC=1 timeout 300 python tools/prof_e2e.py $c > gpurun_out/r2_zc/prof_${c}_nozc.log 2>&1
done
