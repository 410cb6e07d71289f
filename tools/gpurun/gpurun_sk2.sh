mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_out_proj.py -q -x 2>&1 | tail -2 > gpurun_out/sk2.log
timeout 200 python tools/bench_proj.py >> gpurun_out/sk2.log 2>&1
