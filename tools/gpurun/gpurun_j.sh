mkdir -p gpurun_out
for st in 2 3 4; do
  cp variants/libhygen_st$st.so paper_2501_14808_b200/libhygen.so
  timeout 120 python -m pytest tests/test_gpu_parity.py -q -x -k "toy or fuzz1" 2>&1 | tail -1 | sed "s/^/st$st /" >> gpurun_out/v.log
  for c in c1 c2 c3; do timeout 120 python tools/run_config.py $c --time --steps 4 --no-tc 2>&1 | cut -c1-60 | sed "s/^/st$st /" >> gpurun_out/v.log; done
done
