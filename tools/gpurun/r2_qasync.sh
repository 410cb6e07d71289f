# split-K item start-up: Q tile by cp.async beside the first K/V blocks (one latency instead of
# two): parity, per-rank step times, split-K occupancy trace at the 8-way shard
mkdir -p gpurun_out/r2_qasync
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_peer.py -q -x -p no:cacheprovider --timeout 600 > gpurun_out/r2_qasync/tests.log 2>&1
echo rc=$? >> gpurun_out/r2_qasync/tests.log
for r in 1 2; do timeout 300 python tools/exp_tp.py c3 c1 > gpurun_out/r2_qasync/tp_$r.log 2>&1; done
HG_TRACE_TAIL=1 timeout 300 python tools/trace_sk.py c3@8 > gpurun_out/r2_qasync/trace_c3g8.log 2>&1
