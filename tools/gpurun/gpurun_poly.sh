mkdir -p gpurun_out/poly
for m in 0x88 0x00 0xAA 0x80; do
HG_NVCC_DEFS="-DHG_POLY_MASK=$m" python -c "from paper_2501_14808_b200 import build; build.build(force=True)" > /dev/null 2>&1
for c in p1 p2; do HG_HOST_AHEAD=1 timeout 300 python tools/run_config.py $c --time --steps 12 2>&1 | grep "step" | tail -8 > gpurun_out/poly/${c}_$m.log; done
done
