mkdir -p gpurun_out/final2
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3 > gpurun_out/final2/tests.log
timeout 1200 python bench.py > gpurun_out/final2/bench.log 2> gpurun_out/final2/bench.err
echo bench=$? >> gpurun_out/final2/tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final2/smoke.log 2>&1
echo smoke=$? >> gpurun_out/final2/tests.log
