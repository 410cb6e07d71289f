# background append on the tcgen05 CTAs' idle warp (vs the prologue), parity of the fused
# step; cost of the sharded step's exit barrier (1-rank window)
mkdir -p gpurun_out/r2_bg
timeout 300 python tools/exp_tc.py p1 p2 > gpurun_out/r2_bg/exp.log 2>&1
HG_NO_BG_APPEND=1 EXP_TAG=prologue timeout 300 python tools/exp_tc.py p1 p2 >> gpurun_out/r2_bg/exp.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider --timeout 600 \
    -k "fused or whole_tensor or peaked or toy or e2e or prefill_key_split or fuzz" > gpurun_out/r2_bg/tests.log 2>&1
echo rc=$? >> gpurun_out/r2_bg/tests.log
timeout 300 python tools/exp_tp.py c3 > gpurun_out/r2_bg/tp.log 2>&1
HG_TP_EXIT_SKIP=1 EXP_TAG="no-exit " timeout 300 python tools/exp_tp.py c3 >> gpurun_out/r2_bg/tp.log 2>&1
