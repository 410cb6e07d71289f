mkdir -p gpurun_out/check3
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3 > gpurun_out/check3/tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/check3/smoke.log 2>&1
echo smoke=$? >> gpurun_out/check3/tests.log
