mkdir -p gpurun_out
timeout 120 python -m pytest tests/test_gpu_parity.py -q -x -k "toy" > gpurun_out/t0.log 2>&1
echo t0=$? >> gpurun_out/status.txt
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/t.log 2>&1
echo t=$? >> gpurun_out/status.txt
for c in p2 p1 c1 c2 c3; do timeout 120 python tools/run_config.py $c --time --steps 3 2>&1 | cut -c1-80 >> gpurun_out/time.log; done
timeout 600 python bench.py --steps 20 --warmup 5 --no-predictor > gpurun_out/bench.log 2>&1
echo bench=$? >> gpurun_out/status.txt
