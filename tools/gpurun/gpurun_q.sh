mkdir -p gpurun_out
cp paper_2501_14808_b200/libhygen.so /tmp/orig.so
for m in 0x88 0xAA 0x92 0x00; do
  cp variants/libhygen_poly$m.so paper_2501_14808_b200/libhygen.so
  touch paper_2501_14808_b200/libhygen.so
  timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "toy or fuzz1 or p1 or p2 or peaked" 2>&1 | tail -1 | sed "s/^/$m /" >> gpurun_out/q.log
  for c in p1 p2; do timeout 120 python tools/run_config.py $c --time --steps 4 2>&1 | tail -3 | cut -c1-60 | sed "s/^/$m /" >> gpurun_out/q.log; done
done
cp /tmp/orig.so paper_2501_14808_b200/libhygen.so
