mkdir -p gpurun_out
rm -f gpurun_out/w.log
for c in c1 c3; do HG_HOST_AHEAD=1 timeout 120 python tools/run_config.py $c --time --steps 5 2>&1 | tail -4 | cut -c1-110 >> gpurun_out/w.log; done
