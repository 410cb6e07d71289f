mkdir -p gpurun_out/sktma
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "toy or fuzz or full_size or c2" 2>&1 | tail -3 > gpurun_out/sktma/tests.log
for i in 1 2; do
timeout 600 python bench.py --no-predictor > gpurun_out/sktma/b_tma$i.log 2>gpurun_out/sktma/b_tma$i.err
HG_SK_NO_TMA=1 timeout 600 python bench.py --no-predictor > gpurun_out/sktma/b_old$i.log 2>/dev/null
done
