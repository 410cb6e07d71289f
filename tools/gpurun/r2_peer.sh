mkdir -p gpurun_out/r2_peer
export HG_PARITY_LOG=$PWD/gpurun_out/r2_peer/parity.log
timeout 1200 python -m pytest tests/test_gpu_peer.py tests/test_gpu_parity.py -m gpu -q -x -s -p no:cacheprovider -k "peer or peaked or whole" > gpurun_out/r2_peer/tests.log 2>&1
echo rc=$? >> gpurun_out/r2_peer/tests.log
for c in c3@8 c3@4 c3 c1@8 p1 p2; do echo "== $c"; timeout 300 python tools/prof_step.py $c 2>&1 | tail -40; done > gpurun_out/r2_peer/prof.log 2>&1
