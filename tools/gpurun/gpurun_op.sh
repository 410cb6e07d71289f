mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_out_proj.py -q -x 2>&1 | tail -25 > gpurun_out/op.log
