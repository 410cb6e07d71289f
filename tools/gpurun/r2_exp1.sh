mkdir -p gpurun_out/r2_exp1
timeout 600 python tools/exp_shard.py c3@8 c3@4 c3@2 c3 c1@8 c1 > gpurun_out/r2_exp1/exp.log 2>&1
for c in c3@8 c3; do echo "== $c"; timeout 300 python tools/prof_step.py $c 2>&1 | grep -v Warn | tail -12; done > gpurun_out/r2_exp1/prof.log 2>&1
