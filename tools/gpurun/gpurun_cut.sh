mkdir -p gpurun_out/cut2
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "prefill_key_split or e2e or full_size" 2>&1 | tail -3 > gpurun_out/cut2/tests.log
HG_HOST_AHEAD=1 timeout 300 python tools/run_config.py p1 --time --steps 12 2>&1 | grep step | tail -8 > gpurun_out/cut2/p1.log
HG_HOST_AHEAD=1 timeout 300 python tools/run_config.py slow --spec tools/slow_batch_c4_219.pkl --time --steps 12 2>&1 | grep step | tail -8 > gpurun_out/cut2/slow.log
HG_SAVE_SWEEP=gpurun_out/cut2 timeout 900 python bench.py --no-extra > gpurun_out/cut2/bench.log 2> gpurun_out/cut2/bench.err
