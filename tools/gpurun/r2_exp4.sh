mkdir -p gpurun_out/r2_exp4
for w in 1 2 3; do echo "== waves $w"; HG_SK_WAVES=$w EXP_VARIANTS=lpt,lpt_no_tc timeout 600 python tools/exp_shard.py c3@8 c3@4 c3 c1@8 c1 c2; done > gpurun_out/r2_exp4/exp.log 2>&1
