mkdir -p gpurun_out/pf
for c in c1 c1_long c3 c2; do HG_HOST_AHEAD=1 timeout 300 python tools/run_config.py $c --time --steps 10 2>&1 | grep "step" | tail -6 > gpurun_out/pf/$c.log; done
for s in c3_shard_g8 c1_shard_g8; do HG_HOST_AHEAD=1 timeout 300 python tools/run_config.py x --spec tools/$s.pkl --time --steps 10 2>&1 | grep "step" | tail -6 > gpurun_out/pf/$s.log; done
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "full_size or nested or fuzz" 2>&1 | tail -2 > gpurun_out/pf/tests.log
