mkdir -p gpurun_out/waves3
for i in 1 2; do
for w in 4 1; do
HG_SK_WAVES=$w timeout 600 python bench.py --no-predictor > gpurun_out/waves3/b_w${w}_$i.log 2>/dev/null
done
done
