# exp2 split between MUFU and the FMA-pipe polynomial under the power cap (the kernel with
# the tile-0 skip): 0 / 1/8 / 1/4 (default) / 1/2 of the pairs on the polynomial
mkdir -p gpurun_out/r2_poly
V=$PWD/paper_2501_14808_b200/var
for r in 1 2; do
  timeout 300 python tools/exp_tc.py p1 p2 >> gpurun_out/r2_poly/tc.log 2>&1
  for m in 0x00 0x80 0xAA; do HG_SO_OVERRIDE=$V/libhygen_poly$m.so timeout 300 python tools/exp_tc.py p1 p2 >> gpurun_out/r2_poly/tc.log 2>&1; done
done
