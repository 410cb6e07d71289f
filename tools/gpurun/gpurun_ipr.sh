mkdir -p gpurun_out/ipr
for c in c1 c1_long c3; do
  for k in 0 1; do
    if [ $k = 1 ]; then export HG_IPR256_BESIDE_SK=1; else unset HG_IPR256_BESIDE_SK; fi
    timeout 300 python tools/run_config.py $c --time --steps 12 2>&1 | grep step | tail -8 > gpurun_out/ipr/${c}_$k.log
  done
done
