mkdir -p gpurun_out/tpstep
timeout 900 python -m pytest tests/test_gpu_peer.py tests/test_gpu_parity.py -m gpu -q -x -k "peer or world1 or tp" 2>&1 | tail -3 > gpurun_out/tpstep/tests.log
HG_BENCH_SAME_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29555 bench.py --gpus 2 --steps 50 --warmup 5 > gpurun_out/tpstep/bench2.log 2> gpurun_out/tpstep/bench2.err
echo rc=$? >> gpurun_out/tpstep/tests.log
