mkdir -p gpurun_out/check4
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "shard_slices or param_slots" -s 2>&1 | grep -v "^$" | tail -8 > gpurun_out/check4/tests.log
