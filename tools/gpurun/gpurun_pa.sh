mkdir -p gpurun_out/pa
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2 > gpurun_out/pa/tests.log
for i in 1 2; do
timeout 600 python bench.py --no-predictor --no-extra > gpurun_out/pa/b_new$i.log 2>/dev/null
HG_NO_PARAM_APPEND=1 timeout 600 python bench.py --no-predictor --no-extra > gpurun_out/pa/b_old$i.log 2>/dev/null
done
for s in c1_shard_g8; do for k in new old; do
if [ $k = old ]; then export HG_NO_PARAM_APPEND=1; else unset HG_NO_PARAM_APPEND; fi
HG_HOST_AHEAD=1 timeout 300 python tools/run_config.py x --spec tools/$s.pkl --time --steps 12 2>&1 | grep "step" | tail -8 > gpurun_out/pa/${s}_$k.log
HG_HOST_AHEAD=1 timeout 300 python tools/run_config.py c3 --time --steps 12 2>&1 | grep "step" | tail -8 > gpurun_out/pa/c3_$k.log
done; done
