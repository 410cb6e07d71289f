# e2e host step on C3: wall time, device timeline (CUPTI), host phase times; and the ncu
# launch list of the sharded step (C3 8-way shard slice on a 1-rank window)
mkdir -p gpurun_out/r2_e2e
HG_E2E_TRACE=1 timeout 300 python tools/prof_e2e.py c3 > gpurun_out/r2_e2e/prof_c3.log 2> gpurun_out/r2_e2e/prof_c3.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"splitk|tc_attn|combine|append|barrier" \
    --csv --log-file gpurun_out/r2_e2e/launches_tp_c3g8.csv python tools/tp_launches.py c3 8 3 > gpurun_out/r2_e2e/tp_launches.log 2>&1
