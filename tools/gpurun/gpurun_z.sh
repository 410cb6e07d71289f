mkdir -p gpurun_out; rm -f gpurun_out/z.log
cp variants/libhygen_fake.so paper_2501_14808_b200/libhygen.so; touch paper_2501_14808_b200/libhygen.so
for c in p2 p1; do timeout 120 python tools/run_config.py $c --time --steps 3 2>&1 | grep "^p" | cut -c1-80 >> gpurun_out/z.log; done
timeout 120 python tools/trace_tc.py p2 > gpurun_out/z_trace.log 2>&1
