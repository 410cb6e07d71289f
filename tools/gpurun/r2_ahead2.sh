mkdir -p gpurun_out/r2_ahead2
timeout 300 python tools/e2e_ahead.py c3 > gpurun_out/r2_ahead2/c3.log 2>&1
HG_E2E_TRACE=1 timeout 300 python tools/e2e_ahead.py c3 > gpurun_out/r2_ahead2/c3_trace.log 2> gpurun_out/r2_ahead2/c3_trace.err
