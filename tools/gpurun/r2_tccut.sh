# tcgen05 item cuts (greedy LPT with cutting): parity of the tcgen05 paths, then the
# (the item-cut planner was removed after this measurement; HG_NO_TC_CUTS / HG_TC_ITEM_COST are gone -- see git history)
# planner A/B (cuts off / on, item cost 2 / 4 / 8) by CTA end times and event time
mkdir -p gpurun_out/r2_tccut
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider --timeout 600 \
    -k "toy or fuzz or whole_tensor or fused or e2e or peaked or prefill or second_seed or run_to_run" > gpurun_out/r2_tccut/tests.log 2>&1
echo rc=$? >> gpurun_out/r2_tccut/tests.log
for v in "HG_NO_TC_CUTS=1" "HG_TC_ITEM_COST=2" "HG_TC_ITEM_COST=4" "HG_TC_ITEM_COST=8" "HG_NO_TC_CUTS=1 HG_TC_ITEM_COST=1"; do
  env $v timeout 300 python tools/trace_tc_grid.py p1 p2 >> gpurun_out/r2_tccut/grid.log 2>&1
  env $v timeout 300 python tools/exp_tc.py p1 p2 | sed "s/^/$v /" >> gpurun_out/r2_tccut/tc.log 2>&1
done
