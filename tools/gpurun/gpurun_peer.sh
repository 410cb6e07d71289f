mkdir -p gpurun_out/peer
timeout 1200 python -m pytest tests/test_gpu_peer.py tests/test_gpu_parity.py tests/test_gpu_out_proj.py -m gpu -q -x -k "peer or world1 or tp or window or rank" 2>&1 | tail -3 > gpurun_out/peer/tests.log
HG_BENCH_SAME_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29571 bench.py --gpus 4 --steps 20 --warmup 3 > gpurun_out/peer/b4.log 2> gpurun_out/peer/b4.err
echo rc=$? >> gpurun_out/peer/tests.log
