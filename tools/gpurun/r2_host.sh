# host-side cost of a call (validate + plan in one pass over the block table, descriptor image
# assembled in the pinned slot) and the e2e host step on C3; parity of the host-step paths
mkdir -p gpurun_out/r2_host
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider --timeout 600 \
    -k "toy or fuzz or e2e or error or empty or whole_tensor" > gpurun_out/r2_host/tests.log 2>&1
echo rc=$? >> gpurun_out/r2_host/tests.log
for i in 1 2 3; do python tools/plan_time.py; done > gpurun_out/r2_host/plan_time.log 2>&1
HG_E2E_TRACE=1 timeout 300 python tools/prof_e2e.py c3 > gpurun_out/r2_host/prof_c3.log 2> gpurun_out/r2_host/prof_c3.err
