# the final code's GPU suite, smoke, bench line, and the 2-rank bench path on one GPU
mkdir -p gpurun_out/r2_final3
O=gpurun_out/r2_final3
export HG_PARITY_LOG=$PWD/$O/parity.log
timeout 1800 python -m pytest tests -m gpu -q -x -p no:cacheprovider > $O/tests.log 2>&1
echo rc=$? >> $O/tests.log
unset HG_PARITY_LOG
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
echo smoke_rc=$? >> $O/smoke.log
timeout 1500 python bench.py > $O/bench.log 2> $O/bench.err
echo bench_rc=$? >> $O/bench.err
HG_BENCH_SAME_GPU=1 timeout 600 python bench.py --gpus 2 --steps 20 --warmup 3 > $O/bench_g2_samegpu.log 2>&1
echo rc=$? >> $O/bench_g2_samegpu.log
