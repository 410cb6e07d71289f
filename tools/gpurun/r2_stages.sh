# split-K ring depth at the small shards: 2 stages x 3 CTAs/SM (default) vs 3 or 4 stages x 2 CTAs/SM
# (the planner sized for 2 resident CTAs), per-rank step times
mkdir -p gpurun_out/r2_stages
V=$PWD/paper_2501_14808_b200/var
timeout 300 python tools/exp_tp.py c3 c1 > gpurun_out/r2_stages/default.log 2>&1
HG_SO_OVERRIDE=$V/libhygen_s3.so HG_SK_CTAS_PER_SM=2 timeout 300 python tools/exp_tp.py c3 c1 > gpurun_out/r2_stages/s3.log 2>&1
HG_SO_OVERRIDE=$V/libhygen_s4.so HG_SK_CTAS_PER_SM=2 timeout 300 python tools/exp_tp.py c3 c1 > gpurun_out/r2_stages/s4.log 2>&1
HG_SK_CTAS_PER_SM=2 timeout 300 python tools/exp_tp.py c3 c1 > gpurun_out/r2_stages/default_per2.log 2>&1
timeout 300 python tools/exp_tp.py c3 c1 > gpurun_out/r2_stages/default2.log 2>&1
