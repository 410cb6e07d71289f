mkdir -p gpurun_out; rm -f gpurun_out/fc2.log
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "fused_combine or fuzz1 or full_size" 2>&1 | tail -2 > gpurun_out/fc2.log
for c in c1 c2 c3; do timeout 120 python tools/run_config.py $c --time --steps 6 2>&1 | grep "^c" | tail -4 | cut -c1-100 >> gpurun_out/fc2.log; done
