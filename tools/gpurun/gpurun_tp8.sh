mkdir -p gpurun_out/tp8
HG_BENCH_SAME_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 --master-port 29561 bench.py --gpus 8 --steps 20 --warmup 3 > gpurun_out/tp8/bench8.log 2> gpurun_out/tp8/bench8.err
echo rc=$? >> gpurun_out/tp8/bench8.log
HG_BENCH_SAME_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29562 bench.py --gpus 4 --steps 20 --warmup 3 --impl reference > gpurun_out/tp8/ref4.log 2> gpurun_out/tp8/ref4.err
echo rc=$? >> gpurun_out/tp8/ref4.log
