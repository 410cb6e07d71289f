mkdir -p gpurun_out/full
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/full/gpu.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -5 > gpurun_out/full/tests.log
timeout 1200 python bench.py > gpurun_out/full/bench.log 2> gpurun_out/full/bench.err
echo bench=$? >> gpurun_out/full/tests.log
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/full/bench_ref.log 2> gpurun_out/full/bench_ref.err
echo bench_ref=$? >> gpurun_out/full/tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/full/smoke.log 2>&1
echo smoke=$? >> gpurun_out/full/tests.log
