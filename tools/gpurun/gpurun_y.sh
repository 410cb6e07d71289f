mkdir -p gpurun_out; rm -f gpurun_out/y.log
for n in 148 74 37 18; do for c in c1 c1_long c2 c3; do
  HG_TC_CTAS=$n timeout 120 python tools/run_config.py $c --time --steps 4 2>&1 | grep "^c" | tail -3 | cut -c1-100 | sed "s/^/$n /" >> gpurun_out/y.log
done; done
