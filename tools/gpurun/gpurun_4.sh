mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "tp_path or toy or e2e or error" > gpurun_out/t_new.log 2>&1
echo tnew=$? >> gpurun_out/status.txt
timeout 900 python bench.py --steps 20 --warmup 5 --extra > gpurun_out/bench.log 2>&1
echo bench=$? >> gpurun_out/status.txt
