mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "error_leaves" 2>&1 | tail -2 > gpurun_out/n_tests.log
for c in c1 c2 c3 c1_long; do
  timeout 120 python tools/run_config.py $c --time --steps 5 2>&1 | tail -3 | cut -c1-90 | sed "s/^/tc   /" >> gpurun_out/n_time.log
  timeout 120 python tools/run_config.py $c --time --steps 5 --no-tc 2>&1 | tail -3 | cut -c1-90 | sed "s/^/notc /" >> gpurun_out/n_time.log
done
