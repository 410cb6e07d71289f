# folded exit barrier: per-rank cost (vs its own kernel), multi-rank correctness on one GPU
mkdir -p gpurun_out/r2_exit
timeout 300 python tools/exp_tp.py c3 c1 > gpurun_out/r2_exit/tp.log 2>&1
HG_TP_EXIT_KERNEL=1 EXP_TAG="exit-kernel " timeout 300 python tools/exp_tp.py c3 c1 >> gpurun_out/r2_exit/tp.log 2>&1
timeout 900 python -m pytest tests/test_gpu_peer.py tests/test_gpu_out_proj.py -q -x -p no:cacheprovider --timeout 800 > gpurun_out/r2_exit/peer.log 2>&1
echo rc=$? >> gpurun_out/r2_exit/peer.log
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "tp or shard" > gpurun_out/r2_exit/tests.log 2>&1
echo rc=$? >> gpurun_out/r2_exit/tests.log
HG_BENCH_SAME_GPU=1 timeout 600 python bench.py --gpus 4 --steps 20 --warmup 3 --no-extra --no-predictor > gpurun_out/r2_exit/bench_g4_samegpu.log 2>&1
echo rc=$? >> gpurun_out/r2_exit/bench_g4_samegpu.log
