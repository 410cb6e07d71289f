mkdir -p gpurun_out/final
timeout 1200 python bench.py > gpurun_out/final/bench.log 2> gpurun_out/final/bench.err
echo rc=$? >> gpurun_out/final/status.txt
