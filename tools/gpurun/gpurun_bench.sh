mkdir -p gpurun_out/final
timeout 1200 python bench.py --no-predictor > gpurun_out/final/bench_np.log 2> gpurun_out/final/bench_np.err
echo rc=$? >> gpurun_out/final/status.txt
HG_HOST_AHEAD=1 timeout 300 python tools/run_config.py x --spec tools/c3_shard_g8.pkl --time --steps 10 2>&1 | grep "step" | tail -4 > gpurun_out/final/c3g8.log
