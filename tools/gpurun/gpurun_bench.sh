mkdir -p gpurun_out/final
timeout 1200 python bench.py --no-predictor > gpurun_out/final/bench_np.log 2> gpurun_out/final/bench_np.err
echo rc=$? >> gpurun_out/final/status.txt
