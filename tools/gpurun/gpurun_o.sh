mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3 > gpurun_out/o_tests.log
for c in p1 p2 c1 c1_long c3; do timeout 120 python tools/run_config.py $c --time --steps 4 2>&1 | tail -3 | cut -c1-90 | sed "s/^/$c /" >> gpurun_out/o_time.log; done
