# tcgen05: Q tile 0 of a 256-row prefill item stops at its own causal range (one KV tile
# fewer than tile 1): a short guarded smoke first, then parity, then p1 / p2 timing A/B
mkdir -p gpurun_out/r2_tcskip
O=gpurun_out/r2_tcskip
timeout -s KILL 180 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "test_toy" > $O/smoke_tests.log 2>&1
echo rc=$? >> $O/smoke_tests.log
if grep -q "rc=0" $O/smoke_tests.log; then
  timeout -s KILL 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_peer.py -q -x -p no:cacheprovider > $O/tests.log 2>&1
  echo rc=$? >> $O/tests.log
  for r in 1 2; do timeout -s KILL 300 python tools/exp_tc.py p1 p2 >> $O/tc.log 2>&1; done
  timeout -s KILL 300 python tools/trace_tc_grid.py p1 p2 >> $O/grid.log 2>&1
fi
