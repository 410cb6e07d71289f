mkdir -p gpurun_out/r2_exp2
for c in "c3@8" "c3@8 ev" "c1"; do echo "== $c"; timeout 300 python tools/prof_step2.py $c 2>&1 | grep -v Warn | tail -32; done > gpurun_out/r2_exp2/prof.log 2>&1
