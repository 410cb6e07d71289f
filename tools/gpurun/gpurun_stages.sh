mkdir -p gpurun_out/stages
timeout 600 python bench.py --no-predictor --no-extra > gpurun_out/stages/b_s2.log 2>/dev/null
HG_NVCC_DEFS="-DHG_SK_STAGES=3" python -c "from paper_2501_14808_b200 import build; build.build(force=True)" > gpurun_out/stages/build3.log 2>&1
timeout 600 python bench.py --no-predictor --no-extra > gpurun_out/stages/b_s3.log 2>/dev/null
HG_NVCC_DEFS="-DHG_SK_STAGES=4" python -c "from paper_2501_14808_b200 import build; build.build(force=True)" > gpurun_out/stages/build4.log 2>&1
timeout 600 python bench.py --no-predictor --no-extra > gpurun_out/stages/b_s4.log 2>/dev/null
