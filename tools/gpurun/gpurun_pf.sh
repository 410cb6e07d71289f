mkdir -p gpurun_out; rm -f gpurun_out/pf.log
for pf in 0 1 2 4; do
  cp variants/libhygen_pf$pf.so paper_2501_14808_b200/libhygen.so; touch paper_2501_14808_b200/libhygen.so
  timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "toy or fuzz1" 2>&1 | tail -1 | sed "s/^/pf$pf /" >> gpurun_out/pf.log
  for c in c1 c2 c3; do timeout 120 python tools/run_config.py $c --time --steps 6 --no-tc 2>&1 | grep "^c" | tail -4 | cut -c1-75 | sed "s/^/pf$pf /" >> gpurun_out/pf.log; done
done
