mkdir -p gpurun_out
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.log 2>&1
echo bench=$? >> gpurun_out/status.txt
