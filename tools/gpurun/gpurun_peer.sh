mkdir -p gpurun_out/peer
timeout 1200 python -m pytest tests/test_gpu_peer.py -m gpu -q -x 2>&1 | tail -5 > gpurun_out/peer/tests.log
