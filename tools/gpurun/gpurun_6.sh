mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "toy or fuzz or full_size or peaked or variants" > gpurun_out/t.log 2>&1
echo t=$? >> gpurun_out/status.txt
timeout 120 python tools/run_config.py p2 --time --steps 5 > gpurun_out/p2_time.log 2>&1
timeout 120 python tools/run_config.py p1 --time --steps 5 > gpurun_out/p1_time.log 2>&1
timeout 120 python tools/run_config.py c3 --time --steps 3 > gpurun_out/c3_time.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc_attn -s 2 -c 1 -o gpurun_out/prof_p2 python tools/run_config.py p2 --steps 1 > gpurun_out/ncu_p2.log 2>&1
echo done=$? >> gpurun_out/status.txt
