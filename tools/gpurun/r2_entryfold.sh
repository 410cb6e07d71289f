# sharded HBM route: entry barrier in split-K's first CTA and exit barrier in its last (2 launches
# per step: append + split-K) vs barrier kernels; parity of the peer-window paths, per-rank A/B
mkdir -p gpurun_out/r2_entryfold
timeout 1200 python -m pytest tests/test_gpu_peer.py tests/test_gpu_parity.py -q -x -p no:cacheprovider --timeout 600 > gpurun_out/r2_entryfold/tests.log 2>&1
echo rc=$? >> gpurun_out/r2_entryfold/tests.log
for r in 1 2; do
  timeout 300 python tools/exp_tp.py c3 c1 > gpurun_out/r2_entryfold/tp_fold_$r.log 2>&1
  HG_TP_ENTRY_KERNEL=1 HG_TP_EXIT_KERNEL=1 timeout 300 python tools/exp_tp.py c3 c1 > gpurun_out/r2_entryfold/tp_kernels_$r.log 2>&1
done
HG_BENCH_SAME_GPU=1 timeout 600 python bench.py --gpus 2 --steps 20 --warmup 3 > gpurun_out/r2_entryfold/bench_g2_samegpu.log 2>&1
echo rc=$? >> gpurun_out/r2_entryfold/bench_g2_samegpu.log
