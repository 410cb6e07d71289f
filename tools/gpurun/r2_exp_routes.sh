mkdir -p gpurun_out/r2_exp6
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_alloc_e2e.py -q -x -p no:cacheprovider > gpurun_out/r2_exp6/tests.log 2>&1
echo rc=$? >> gpurun_out/r2_exp6/tests.log
EXP_VARIANTS=default,tc_route,no_prefix timeout 900 python tools/exp_shard.py c3@8 c3@4 c3@2 c3 c1@8 c1 c2 c2_nested p1 p2 > gpurun_out/r2_exp6/exp.log 2>&1
