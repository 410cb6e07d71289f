# split-K in-kernel merge (no combine kernel on the HBM route) and tcgen05 item cuts: parity + A/B
# (the item-cut planner was removed after this measurement; HG_NO_TC_CUTS / HG_TC_ITEM_COST are gone -- see git history)
mkdir -p gpurun_out/r2_skmerge
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_peer.py -q -x -p no:cacheprovider --timeout 600 \
    > gpurun_out/r2_skmerge/tests.log 2>&1
echo rc=$? >> gpurun_out/r2_skmerge/tests.log
timeout 300 python tools/exp_tp.py c3 c1 > gpurun_out/r2_skmerge/tp.log 2>&1
HG_NO_SK_MERGE=1 timeout 300 python tools/exp_tp.py c3 c1 > gpurun_out/r2_skmerge/tp_nomerge.log 2>&1
timeout 300 python tools/exp_tp.py c3 c1 > gpurun_out/r2_skmerge/tp2.log 2>&1
for c in c3@8 c1@8; do HG_TRACE_TAIL=1 timeout 300 python tools/trace_sk.py $c; done > gpurun_out/r2_skmerge/trace_tail.log 2>&1
timeout 300 python tools/exp_tc.py p1 p2 > gpurun_out/r2_skmerge/tc.log 2>&1
HG_NO_TC_CUTS=1 timeout 300 python tools/exp_tc.py p1 p2 > gpurun_out/r2_skmerge/tc_nocuts.log 2>&1
timeout 300 python tools/exp_tc.py p1 p2 > gpurun_out/r2_skmerge/tc2.log 2>&1
