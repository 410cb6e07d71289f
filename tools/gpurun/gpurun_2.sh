mkdir -p gpurun_out
timeout 400 python bench.py --steps 10 --warmup 3 --extra > gpurun_out/bench.log 2>&1
echo bench=$? >> gpurun_out/status.txt
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --profile > gpurun_out/ncu_launch.log 2>&1
echo ncu=$? >> gpurun_out/status.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:splitk -s 5 -c 1 -o gpurun_out/prof_splitk python bench.py --steps 2 --warmup 3 --profile > gpurun_out/ncu_full.log 2>&1
echo ncufull=$? >> gpurun_out/status.txt
