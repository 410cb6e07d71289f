# quick health check of HEAD: single-GPU suite (peer tests last), the default bench line
mkdir -p gpurun_out/r2_chk
export HG_PARITY_LOG=$PWD/gpurun_out/r2_chk/parity.log
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/r2_chk/gpu.txt
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider --timeout 600 \
    --ignore=tests/test_gpu_peer.py > gpurun_out/r2_chk/tests.log 2>&1
echo rc=$? >> gpurun_out/r2_chk/tests.log
timeout 900 python bench.py > gpurun_out/r2_chk/bench.log 2> gpurun_out/r2_chk/bench.err
echo bench_rc=$? >> gpurun_out/r2_chk/bench.err
timeout 900 python -m pytest tests/test_gpu_peer.py -x -q -p no:cacheprovider --timeout 800 > gpurun_out/r2_chk/peer.log 2>&1
echo rc=$? >> gpurun_out/r2_chk/peer.log
