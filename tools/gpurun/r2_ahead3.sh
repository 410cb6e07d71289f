timeout 300 python tools/e2e_ahead_prof.py c3 > gpurun_out/r2_ahead2/prof.log 2>&1
