# full GPU suite; whole-tensor parity lines logged for profiles/r2/parity_full_size.log
mkdir -p gpurun_out/r2_tests
export HG_PARITY_LOG=$PWD/gpurun_out/r2_tests/parity.log
timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider --durations=25 > gpurun_out/r2_tests/tests.log 2>&1
echo rc=$? >> gpurun_out/r2_tests/tests.log
