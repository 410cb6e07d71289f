mkdir -p gpurun_out/app
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "append or fused or e2e or toy or fuzz" 2>&1 | tail -2 > gpurun_out/app/tests.log
timeout 300 python tools/prof_step.py c1 > gpurun_out/app/prof_c1.log 2>&1
for s in c1_shard_g8; do HG_HOST_AHEAD=1 timeout 300 python tools/run_config.py x --spec tools/$s.pkl --time --steps 10 2>&1 | grep "step" | tail -6 > gpurun_out/app/$s.log; done
HG_HOST_AHEAD=1 timeout 300 python tools/run_config.py c1 --time --steps 10 2>&1 | grep "step" | tail -6 > gpurun_out/app/c1.log
