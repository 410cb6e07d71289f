# split-K grid sizing at the 8-way shard: waves of LPT pieces (1 / 1.25 / 1.5 / 2), CTA end
# spread by SM, per-rank step time
mkdir -p gpurun_out/r2_skwaves
for w in 1 1.25 1.5 2; do
  HG_SK_WAVES=$w HG_TRACE_TAIL=1 timeout 300 python tools/trace_sk.py c3@8 > gpurun_out/r2_skwaves/trace_$w.log 2>&1
  HG_SK_WAVES=$w timeout 300 python tools/exp_tp.py c3 c1 > gpurun_out/r2_skwaves/tp_$w.log 2>&1
done
