# tcgen05: per-tile QREADY / OFREE: the next item's tile 0 starts while tile 1 is in its epilogue
# guarded smoke, parity, p1 / p2 A/B against the previous kernel (var/libhygen_prev.so)
mkdir -p gpurun_out/r2_qready
O=gpurun_out/r2_qready
timeout -s KILL 180 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "test_toy" > $O/smoke_tests.log 2>&1
echo rc=$? >> $O/smoke_tests.log
if grep -q "rc=0" $O/smoke_tests.log; then
  timeout -s KILL 1500 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider > $O/tests.log 2>&1
  echo rc=$? >> $O/tests.log
  for r in 1 2; do
    timeout -s KILL 300 python tools/exp_tc.py p1 p2 >> $O/tc.log 2>&1
    HG_SO_OVERRIDE=$PWD/paper_2501_14808_b200/var/libhygen_prev.so timeout -s KILL 300 python tools/exp_tc.py p1 p2 >> $O/tc.log 2>&1
  done
fi
