mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/t.log 2>&1
echo t=$? >> gpurun_out/status.txt
