mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3 > gpurun_out/k_tests.log
for c in p1 p2 c1 c2 c3; do timeout 120 python tools/run_config.py $c --time --steps 5 2>&1 | tail -6 | sed "s/^/$c /" >> gpurun_out/k_time.log; done
