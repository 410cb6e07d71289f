mkdir -p gpurun_out/r2_exp5
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "variants or nested_full or gqa or fuzz or whole or prefix_group or e2e" > gpurun_out/r2_exp5/tests.log 2>&1
echo rc=$? >> gpurun_out/r2_exp5/tests.log
EXP_VARIANTS=default,tc_route,hbm_route,no_prefix timeout 900 python tools/exp_shard.py c3@8 c3@4 c3@2 c3 c1@8 c1 c2 c2_nested c1_long p1 p2 > gpurun_out/r2_exp5/exp.log 2>&1
