# full GPU suite, smoke, the default bench line, and the multi-rank bench path as a
# same-GPU functional run (self-launch under torch.distributed.run)
mkdir -p gpurun_out/r2_full
export HG_PARITY_LOG=$PWD/gpurun_out/r2_full/parity.log
timeout 1800 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/r2_full/tests.log 2>&1
echo rc=$? >> gpurun_out/r2_full/tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_full/smoke.log 2>&1
echo smoke_rc=$? >> gpurun_out/r2_full/smoke.log
timeout 1500 python bench.py > gpurun_out/r2_full/bench.log 2> gpurun_out/r2_full/bench.err
echo bench_rc=$? >> gpurun_out/r2_full/bench.err
HG_BENCH_SAME_GPU=1 timeout 600 python bench.py --gpus 2 --steps 20 --warmup 3 > gpurun_out/r2_full/bench_g2_samegpu.log 2>&1
echo rc=$? >> gpurun_out/r2_full/bench_g2_samegpu.log
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2_full/bench_ref.log 2>&1
