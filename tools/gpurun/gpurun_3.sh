mkdir -p gpurun_out
timeout 120 python -m pytest tests/test_gpu_parity.py -x -q -k "toy and not peaked" > gpurun_out/t_toy.log 2>&1
echo toy=$? >> gpurun_out/status.txt
timeout 600 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1
echo pytest=$? >> gpurun_out/status.txt
timeout 400 python bench.py --steps 20 --warmup 5 --extra > gpurun_out/bench.log 2>&1
echo bench=$? >> gpurun_out/status.txt
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"splitk|tc_attn|combine|append" --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --profile > gpurun_out/ncu_launch.log 2>&1
echo ncu=$? >> gpurun_out/status.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"splitk|tc_attn" -s 2 -c 2 -o gpurun_out/prof_c1 python bench.py --steps 2 --warmup 3 --profile > gpurun_out/ncu_full.log 2>&1
echo ncufull=$? >> gpurun_out/status.txt
