mkdir -p gpurun_out; rm -f gpurun_out/pdl2.log
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2 > gpurun_out/pdl2.log
for c in c1 c1_long c2 c3; do
  timeout 120 python tools/run_config.py $c --time --steps 6 2>&1 | grep "^c" | tail -4 | cut -c1-80 | sed "s/^/fused /" >> gpurun_out/pdl2.log
  timeout 120 python tools/run_config.py $c --time --steps 6 --sepcomb 2>&1 | grep "^c" | tail -4 | cut -c1-80 | sed "s/^/sep   /" >> gpurun_out/pdl2.log
done
timeout 200 python tools/prof_step.py c3 > gpurun_out/prof_c3.log 2>&1
