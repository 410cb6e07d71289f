mkdir -p gpurun_out/r2_reg
for v in "" R224 R192; do
  if [ -n "$v" ]; then export HG_SO_OVERRIDE=$PWD/paper_2501_14808_b200/var/libhygen_$v.so; else unset HG_SO_OVERRIDE; fi
  timeout 300 python tools/exp_tc.py p1 p2 >> gpurun_out/r2_reg/exp.log 2>&1
done
unset HG_SO_OVERRIDE
timeout 300 python tools/trace_tc.py p2 > gpurun_out/r2_reg/trace_p2.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "toy or whole_tensor or peaked or fuzz" > gpurun_out/r2_reg/tests.log 2>&1; echo rc=$? >> gpurun_out/r2_reg/tests.log
