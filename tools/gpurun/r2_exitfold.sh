# sharded HBM route: exit barrier in split-K's last CTA (folded) vs its own kernel; parity of the
# peer-window paths, per-rank step A/B, split-K CTA durations by SM
mkdir -p gpurun_out/r2_exitfold
timeout 1200 python -m pytest tests/test_gpu_peer.py tests/test_gpu_parity.py -q -x -p no:cacheprovider --timeout 600 > gpurun_out/r2_exitfold/tests.log 2>&1
echo rc=$? >> gpurun_out/r2_exitfold/tests.log
for r in 1 2; do
  timeout 300 python tools/exp_tp.py c3 c1 > gpurun_out/r2_exitfold/tp_fold_$r.log 2>&1
  HG_TP_EXIT_KERNEL=1 timeout 300 python tools/exp_tp.py c3 c1 > gpurun_out/r2_exitfold/tp_kernel_$r.log 2>&1
done
HG_TRACE_TAIL=1 timeout 300 python tools/trace_sk.py c3@8 > gpurun_out/r2_exitfold/trace_c3g8.log 2>&1
