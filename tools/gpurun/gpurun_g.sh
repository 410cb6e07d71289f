mkdir -p gpurun_out
for sp in 0 1024 2048 3072 4096 8192; do timeout 120 python tools/run_config.py c1 --time --steps 4 --split $sp 2>&1 | cut -c1-75 >> gpurun_out/split.log; done
for sp in 0 2048 4096 8192; do timeout 120 python tools/run_config.py c2 --time --steps 3 --split $sp 2>&1 | cut -c1-75 >> gpurun_out/split.log; done
for sp in 0 2048 4096 8192; do timeout 120 python tools/run_config.py c3 --time --steps 3 --split $sp 2>&1 | cut -c1-75 >> gpurun_out/split.log; done
