mkdir -p gpurun_out/combside
for i in 1 2; do
timeout 600 python bench.py --no-predictor > gpurun_out/combside/b_base$i.log 2>/dev/null
HG_COMB_SIDE=1 timeout 600 python bench.py --no-predictor > gpurun_out/combside/b_side$i.log 2>/dev/null
done
