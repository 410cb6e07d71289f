mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc_attn -s 2 -c 1 -o gpurun_out/tc_p2 python tools/run_config.py p2 --steps 1 > gpurun_out/s_ncu.log 2>&1
ls -la gpurun_out/ >> gpurun_out/s_ncu.log
