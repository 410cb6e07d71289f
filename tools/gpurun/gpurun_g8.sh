mkdir -p gpurun_out/g8c
for w in 4 2 1; do
export HG_SK_WAVES=$w
HG_HOST_AHEAD=1 timeout 300 python tools/run_config.py x --spec tools/c1_shard_g8.pkl --time --steps 10 2>&1 | grep "step" | tail -6 > gpurun_out/g8c/g8_w$w.log
for c in c1 c2 c3; do HG_HOST_AHEAD=1 timeout 300 python tools/run_config.py $c --time --steps 10 2>&1 | grep "step" | tail -6 > gpurun_out/g8c/${c}_w$w.log; done
done
