mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none -k regex:out_proj -s 3 -c 1 -o gpurun_out/gemm python tools/bench_proj.py 768 8192 8192 > gpurun_out/gemm_ncu.log 2>&1
