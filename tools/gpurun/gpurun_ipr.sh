mkdir -p gpurun_out/ipr2
for c in c1 c1_long c3; do
  for k in base hi hi256; do
    unset HG_TC_HI HG_IPR256_BESIDE_SK
    if [ $k = hi ]; then export HG_TC_HI=1; fi
    if [ $k = hi256 ]; then export HG_TC_HI=1 HG_IPR256_BESIDE_SK=1; fi
    HG_HOST_AHEAD=1 timeout 300 python tools/run_config.py $c --time --steps 16 2>&1 | grep step | tail -12 > gpurun_out/ipr2/${c}_$k.log
  done
done
