mkdir -p gpurun_out; rm -f gpurun_out/ipr.log
for v in 0 1; do for c in c1 c1_long c3; do
  HG_IPR256=$v timeout 120 python tools/run_config.py $c --time --steps 8 2>&1 | grep "^c" | tail -6 | cut -c1-80 | sed "s/^/ipr256=$v /" >> gpurun_out/ipr.log
done; done
