mkdir -p gpurun_out; rm -f gpurun_out/san*.log
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_rope.py -q -x -k "toy or fuzz_rope and 1" > gpurun_out/san_rope.log 2>&1; echo rope=$? >> gpurun_out/san.log
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_out_proj.py -q -x -k "single_rank" > gpurun_out/san_proj.log 2>&1; echo proj=$? >> gpurun_out/san.log
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_peer.py -q -x -k "world1" > gpurun_out/san_peer.log 2>&1; echo peer=$? >> gpurun_out/san.log
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -q -x -k "nested_fuzz and (0 or 1 or 2)" > gpurun_out/san_nested.log 2>&1; echo nested=$? >> gpurun_out/san.log
timeout 900 compute-sanitizer --tool racecheck --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -q -x -k "toy_a and 0 and 1.0" > gpurun_out/san_race.log 2>&1; echo race=$? >> gpurun_out/san.log
