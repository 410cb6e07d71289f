mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "fused_combine" 2>&1 | tail -5 > gpurun_out/fc.log
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3 >> gpurun_out/fc.log
for c in c1 c2 c3; do timeout 120 python tools/run_config.py $c --time --steps 5 2>&1 | grep "^c" | tail -3 | cut -c1-100 >> gpurun_out/fc.log; done
timeout 200 python tools/prof_step.py c3 > gpurun_out/prof_c3.log 2>&1
