mkdir -p gpurun_out
timeout 120 python tools/trace_tc.py p2 > gpurun_out/r_trace_p2.log 2>&1
timeout 120 python tools/trace_tc.py p1 > gpurun_out/r_trace_p1.log 2>&1
