# the device-side invariant checks (HG_DCHECK, built with -DHG_CHECKS: index ranges of Q /
# partial slots / merged rows, per-token arrival counts of the in-kernel merge, the exit
# ticket) over the whole GPU parity and peer suites -- compute-sanitizer is closed on this
# pool, so the kernels check themselves
mkdir -p gpurun_out/r2_checks
export HG_SO_OVERRIDE=$PWD/paper_2501_14808_b200/var/libhygen_checks.so
python -c "import paper_2501_14808_b200 as hg; print(\"loaded\", hg.SO_PATH)" > gpurun_out/r2_checks/tests.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider >> gpurun_out/r2_checks/tests.log 2>&1
echo rc=$? >> gpurun_out/r2_checks/tests.log
grep -c "HG_DCHECK failed" gpurun_out/r2_checks/tests.log >> gpurun_out/r2_checks/tests.log
