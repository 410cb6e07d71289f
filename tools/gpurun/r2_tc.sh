# tcgen05 prefill kernel: parity of the fused-append path, then the A/B decomposition
# (default / no K-V traffic / no softmax) and CTA 0's per-KV-tile timeline on p2
mkdir -p gpurun_out/r2_tc
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider --timeout 600 \
    -k "toy or fuzz or whole_tensor or fused or e2e" > gpurun_out/r2_tc/tests.log 2>&1
echo rc=$? >> gpurun_out/r2_tc/tests.log
for v in "" NOLOAD NOSOFTMAX; do
  if [ -n "$v" ]; then export HG_SO_OVERRIDE=$PWD/paper_2501_14808_b200/var/libhygen_$v.so; else unset HG_SO_OVERRIDE; fi
  timeout 300 python tools/exp_tc.py p1 p2 >> gpurun_out/r2_tc/exp.log 2>&1
done
unset HG_SO_OVERRIDE
timeout 300 python tools/trace_tc.py p2 > gpurun_out/r2_tc/trace_p2.log 2>&1
