mkdir -p gpurun_out/e2e
timeout 300 python tools/prof_e2e.py c1 > gpurun_out/e2e/prof_pipe.log 2>&1
HG_E2E_SERIAL=1 timeout 300 python tools/prof_e2e.py c1 > gpurun_out/e2e/prof_serial.log 2>&1
timeout 300 python tools/prof_e2e.py c1 > gpurun_out/e2e/prof_pipe2.log 2>&1
nproc > gpurun_out/e2e/host.txt; lscpu | head -20 >> gpurun_out/e2e/host.txt; nvidia-smi topo -m >> gpurun_out/e2e/host.txt 2>&1
