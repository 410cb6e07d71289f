mkdir -p gpurun_out/clk
for c in p2 p1 c1 c2; do timeout 300 python tools/clock_probe.py $c 3 >> gpurun_out/clk/probe.log 2>&1; done
