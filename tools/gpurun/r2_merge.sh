# split-K merge without smem bank conflicts: parity + per-rank step times + ncu conflicts on c3@8
mkdir -p gpurun_out/r2_merge
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider --timeout 600 \
    -k "toy or fuzz or whole_tensor or gqa or head_dim or plan_variants or shard or nested" > gpurun_out/r2_merge/tests.log 2>&1
echo rc=$? >> gpurun_out/r2_merge/tests.log
timeout 300 python tools/exp_tp.py c3 c1 > gpurun_out/r2_merge/tp.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,dram__bytes_read.sum \
    --clock-control none -k regex:splitk -c 2 -s 3 python tools/run_config.py c3@8 --steps 5 > gpurun_out/r2_merge/ncu_c3g8.txt 2>&1
