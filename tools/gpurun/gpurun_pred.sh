mkdir -p gpurun_out/pred
HG_SAVE_SWEEP=gpurun_out/pred timeout 900 python bench.py --no-extra > gpurun_out/pred/bench.log 2> gpurun_out/pred/bench.err
