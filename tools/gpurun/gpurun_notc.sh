mkdir -p gpurun_out/notc2
for c in c3 c2 c2_nested c2_g8; do
HG_HOST_AHEAD=1 timeout 300 python tools/run_config.py $c --time --steps 10 2>&1 | grep "step" | tail -6 > gpurun_out/notc2/${c}_tc.log
HG_HOST_AHEAD=1 timeout 300 python tools/run_config.py $c --time --steps 10 --no-prefix 2>&1 | grep "step" | tail -6 > gpurun_out/notc2/${c}_nopre.log
done
for s in c3_shard_g8; do
HG_HOST_AHEAD=1 timeout 300 python tools/run_config.py x --spec tools/$s.pkl --time --steps 10 --no-prefix 2>&1 | grep "step" | tail -6 > gpurun_out/notc2/${s}_nopre.log
done
