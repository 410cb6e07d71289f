# sharded HBM route: the append's device count instead of a stream join (exit barrier PDL chain)
mkdir -p gpurun_out/r2_join
timeout 300 python tools/exp_tp.py c3 c1 > gpurun_out/r2_join/tp.log 2>&1
HG_TP_APPEND_JOIN=1 EXP_TAG="stream-join " timeout 300 python tools/exp_tp.py c3 c1 >> gpurun_out/r2_join/tp.log 2>&1
timeout 900 python -m pytest tests/test_gpu_peer.py -q -x -p no:cacheprovider --timeout 800 > gpurun_out/r2_join/peer.log 2>&1
echo rc=$? >> gpurun_out/r2_join/peer.log
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "tp or shard or fused" > gpurun_out/r2_join/tests.log 2>&1
echo rc=$? >> gpurun_out/r2_join/tests.log
