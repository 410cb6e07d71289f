mkdir -p gpurun_out/tp2
HG_BENCH_SAME_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 20 --warmup 3 > gpurun_out/tp2/b.log 2> gpurun_out/tp2/b.err
echo rc=$? >> gpurun_out/tp2/b.log
