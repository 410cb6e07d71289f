mkdir -p gpurun_out/psplit
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "prefill_key_split" -s 2>&1 | grep -v "^$" | tail -25 > gpurun_out/psplit/tests.log
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -4 > gpurun_out/psplit/all.log
HG_SAVE_SWEEP=gpurun_out/psplit timeout 900 python bench.py --no-extra > gpurun_out/psplit/bench.log 2> gpurun_out/psplit/bench.err
