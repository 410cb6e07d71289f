mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2 > gpurun_out/p_tests.log
for c in c1 c1_long c2 c3; do timeout 120 python tools/run_config.py $c --time --steps 5 2>&1 | tail -4 | cut -c1-90 | sed "s/^/$c /" >> gpurun_out/p_time.log; done
