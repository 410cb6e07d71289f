mkdir -p gpurun_out/comb
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3 > gpurun_out/comb/tests.log
for c in c1 c3 c2; do HG_HOST_AHEAD=1 timeout 300 python tools/run_config.py $c --time --steps 12 2>&1 | grep step | tail -8 > gpurun_out/comb/$c.log; done
