mkdir -p gpurun_out/peer2
timeout 1200 python -m pytest tests/test_gpu_peer.py tests/test_gpu_parity.py -m gpu -q -x -k "peer or world1 or tp or window or rank or e2e or fused" 2>&1 | tail -3 > gpurun_out/peer2/tests.log
HG_BENCH_SAME_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29581 bench.py --gpus 2 --steps 20 --warmup 3 > gpurun_out/peer2/b2.log 2> gpurun_out/peer2/b2.err
echo rc=$? >> gpurun_out/peer2/tests.log
