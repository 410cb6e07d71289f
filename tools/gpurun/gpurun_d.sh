mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "max_context or gqa_group or head_dim_64 or prefix_group_with or run_to_run" > gpurun_out/t.log 2>&1
echo t=$? >> gpurun_out/status.txt
timeout 600 python bench.py --steps 20 --warmup 5 --no-extra --no-predictor > gpurun_out/bench.log 2>&1
echo bench=$? >> gpurun_out/status.txt
