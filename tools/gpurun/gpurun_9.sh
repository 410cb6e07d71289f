mkdir -p gpurun_out
timeout 120 python -m pytest tests/test_gpu_parity.py -q -x -k "toy" > gpurun_out/t0.log 2>&1
echo t0=$? >> gpurun_out/status.txt
timeout 200 python tools/trace_tc.py p2 > gpurun_out/trace.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "fuzz or full_size or peaked or variants or shared or tp" > gpurun_out/t.log 2>&1
echo t=$? >> gpurun_out/status.txt
for c in p2 p1 c1 c3; do timeout 120 python tools/run_config.py $c --time --steps 3 >> gpurun_out/time.log 2>&1; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc_attn -s 2 -c 1 -o gpurun_out/prof_p2 python tools/run_config.py p2 --steps 1 > gpurun_out/ncu_p2.log 2>&1
