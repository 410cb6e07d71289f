mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/t.log 2>&1
echo t=$? >> gpurun_out/status.txt
for c in c1 c2 c3; do timeout 120 python tools/run_config.py $c --time --steps 3 >> gpurun_out/time.log 2>&1; done
timeout 600 python bench.py --steps 20 --warmup 5 --no-extra --no-predictor > gpurun_out/bench.log 2>&1
echo bench=$? >> gpurun_out/status.txt
for tool in memcheck racecheck synccheck; do
  timeout 600 compute-sanitizer --tool $tool --error-exitcode 9 python tools/run_config.py toy_a --steps 1 > gpurun_out/san_$tool.log 2>&1
  echo san_$tool=$? >> gpurun_out/status.txt
done
timeout 600 compute-sanitizer --tool memcheck --error-exitcode 9 python tools/run_config.py toy_b --steps 1 > gpurun_out/san_memcheck_b.log 2>&1
echo san_memcheck_b=$? >> gpurun_out/status.txt
