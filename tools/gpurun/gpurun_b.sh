mkdir -p gpurun_out
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.log 2>&1
echo bench=$? >> gpurun_out/status.txt
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"splitk|tc_attn|combine|append" --csv --log-file gpurun_out/launches_c1.csv python bench.py --steps 3 --warmup 3 --profile --no-extra > gpurun_out/ncu_launch.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"splitk|tc_attn" -s 2 -c 2 -o gpurun_out/prof_c1 python bench.py --steps 2 --warmup 3 --profile --no-extra > gpurun_out/ncu_full.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc_attn -s 2 -c 1 -o gpurun_out/prof_p2 python tools/run_config.py p2 --steps 1 > gpurun_out/ncu_p2.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:splitk -s 2 -c 1 -o gpurun_out/prof_c2 python tools/run_config.py c2 --steps 1 > gpurun_out/ncu_c2.log 2>&1
echo done=$? >> gpurun_out/status.txt
