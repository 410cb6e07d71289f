mkdir -p gpurun_out/pretc
for k in new old; do
if [ $k = old ]; then export HG_PREFILL_TC_ALWAYS=1; else unset HG_PREFILL_TC_ALWAYS; fi
for c in c1 c1_long c3; do HG_HOST_AHEAD=1 timeout 300 python tools/run_config.py $c --time --steps 12 2>&1 | grep "step" | tail -8 > gpurun_out/pretc/${c}_$k.log; done
for s in c1_shard_g8 c3_shard_g8; do HG_HOST_AHEAD=1 timeout 300 python tools/run_config.py x --spec tools/$s.pkl --time --steps 12 2>&1 | grep "step" | tail -8 > gpurun_out/pretc/${s}_$k.log; done
done
unset HG_PREFILL_TC_ALWAYS
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x 2>&1 | tail -2 > gpurun_out/pretc/tests.log
