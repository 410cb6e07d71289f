mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_peer.py -q -x -s 2>&1 | tail -15 > gpurun_out/l_peer.log
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3 > gpurun_out/l_tests.log
