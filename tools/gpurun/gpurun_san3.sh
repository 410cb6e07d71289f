mkdir -p gpurun_out/san3; rm -f gpurun_out/san3/*.log
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -q -x -k "(test_toy and 0 and 1.0) or (test_fuzz and (1 or 7)) or tp_path" > gpurun_out/san3/param_append.log 2>&1; echo memcheck=$? >> gpurun_out/san3/status.log
timeout 900 compute-sanitizer --tool racecheck --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -q -x -k "test_toy and toy_a and 0 and 1.0" > gpurun_out/san3/race.log 2>&1; echo racecheck=$? >> gpurun_out/san3/status.log
