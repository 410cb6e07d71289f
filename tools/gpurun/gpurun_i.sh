mkdir -p gpurun_out
for o in 0 1; do for c in c1 c2 c3; do HG_SPLITK_FIRST=$o timeout 120 python tools/run_config.py $c --time --steps 4 2>&1 | cut -c1-60 | sed "s/^/order$o /" >> gpurun_out/order.log; done; done
for o in 0 1; do HG_SPLITK_FIRST=$o timeout 300 python bench.py --steps 30 --warmup 5 --no-predictor --no-extra 2>&1 | python3 -c "import json,sys; d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); print('order', $o, d['ms_per_step'], d['step_breakdown_ms'])" >> gpurun_out/order.log; done
