mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "nested" 2>&1 | tail -15 > gpurun_out/m_nested.log
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3 > gpurun_out/m_tests.log
for c in c2 c2_nested c2_g8; do timeout 120 python tools/run_config.py $c --time --steps 4 2>&1 | tail -2 | cut -c1-200 | sed "s/^/$c /" >> gpurun_out/m_time.log; done
