set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
echo smoke=$? >> gpurun_out/status.txt
timeout 900 python -m pytest tests -m gpu -x -q -k "not fuzz" > gpurun_out/pytest_gpu.log 2>&1
echo pytest=$? >> gpurun_out/status.txt
timeout 600 python -m pytest tests -m gpu -q -k "fuzz" > gpurun_out/pytest_fuzz.log 2>&1
echo fuzz=$? >> gpurun_out/status.txt
timeout 400 python bench.py --steps 10 --warmup 3 --extra > gpurun_out/bench.log 2>&1
echo bench=$? >> gpurun_out/status.txt
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --profile > gpurun_out/ncu_launch.log 2>&1
echo ncu=$? >> gpurun_out/status.txt
