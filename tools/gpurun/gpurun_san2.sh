mkdir -p gpurun_out/san2; rm -f gpurun_out/san2/*.log
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -q -x -k "prefill_key_split and (gqa5 or mha_64rows or short_ctx)" > gpurun_out/san2/split.log 2>&1; echo split=$? >> gpurun_out/san2/status.log
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -q -x -k "e2e and (toy_a or toy_b or interleaved or d64 or errors)" > gpurun_out/san2/e2e.log 2>&1; echo e2e=$? >> gpurun_out/san2/status.log
timeout 900 compute-sanitizer --tool racecheck --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -q -x -k "prefill_key_split and gqa5" > gpurun_out/san2/race.log 2>&1; echo race=$? >> gpurun_out/san2/status.log
