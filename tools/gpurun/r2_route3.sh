# route 3 (prefill on tcgen05 tiles, prefix nodes on split-K, split-K merging every partial):
# full parity file, then the host step's e2e A/B against route 1 (HG_E2E_NODES_TC)
mkdir -p gpurun_out/r2_route3
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider --timeout 600 > gpurun_out/r2_route3/tests.log 2>&1
echo rc=$? >> gpurun_out/r2_route3/tests.log
for c in c3 c1; do
  HG_E2E_TRACE=1 timeout 300 python tools/prof_e2e.py $c > gpurun_out/r2_route3/prof_$c.log 2> gpurun_out/r2_route3/prof_$c.err
  HG_E2E_NODES_TC=1 timeout 300 python tools/prof_e2e.py $c > gpurun_out/r2_route3/prof_${c}_route1.log 2>&1
done
