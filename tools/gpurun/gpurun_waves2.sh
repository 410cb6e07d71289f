mkdir -p gpurun_out/waves2
for i in 1 2; do
timeout 600 python bench.py --no-extra --no-predictor > gpurun_out/waves2/b_base$i.log 2>/dev/null
HG_STEP_WAVES=1 timeout 600 python bench.py --no-extra --no-predictor > gpurun_out/waves2/b_waves$i.log 2>/dev/null
done
