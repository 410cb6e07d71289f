mkdir -p gpurun_out/r2_exp3
timeout 900 python tools/exp_shard.py c3@8 c3@4 c3 c1@8 c1 c2 c1_long p1 > gpurun_out/r2_exp3/exp.log 2>&1
