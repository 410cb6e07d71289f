mkdir -p gpurun_out; rm -f gpurun_out/pdl3.log
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "toy or fuzz1 or full_size" 2>&1 | tail -1 >> gpurun_out/pdl3.log
HG_PDL=1 timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "toy or fuzz1 or full_size" 2>&1 | tail -1 >> gpurun_out/pdl3.log
for cfg in "0 0" "1 0" "1 64" "1 40" "1 24" "0 40"; do set -- $cfg
  for c in c1 c1_long c2 c3; do
    HG_PDL=$1 HG_TC_CTAS=$2 timeout 120 python tools/run_config.py $c --time --steps 8 2>&1 | grep "^c" | tail -6 | awk -v p=$1 -v n=$2 '{print "pdl="p" ctas="n" "$1" "$5}' >> gpurun_out/pdl3.log
  done
done
