mkdir -p gpurun_out/r2_ncu1
ncu --set full --clock-control none -k regex:splitk -c 1 -s 2 -o gpurun_out/r2_ncu1/c3g8_sk python tools/run_config.py c3@8 --no-tc --lpt --steps 3 > gpurun_out/r2_ncu1/ncu.log 2>&1
ncu --set full --clock-control none -k regex:splitk -c 1 -s 2 -o gpurun_out/r2_ncu1/c3_sk python tools/run_config.py c3 --no-tc --lpt --steps 3 >> gpurun_out/r2_ncu1/ncu.log 2>&1
