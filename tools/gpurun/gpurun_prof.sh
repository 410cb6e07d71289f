# Profile refresh: bench JSON line, ncu launch list of the bench command, ncu --set full captures.
mkdir -p gpurun_out/prof
timeout 1200 python bench.py > gpurun_out/prof/bench.log 2>gpurun_out/prof/bench.err
echo bench=$? >> gpurun_out/prof/status.txt
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"splitk|tc_attn|combine|append" --csv --log-file gpurun_out/prof/launches_c1.csv python bench.py --steps 3 --warmup 3 --profile --no-extra > gpurun_out/prof/ncu_launch.log 2>&1
echo launch=$? >> gpurun_out/prof/status.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"splitk|tc_attn" -s 2 -c 2 -o gpurun_out/prof/c1 python bench.py --steps 2 --warmup 3 --profile --no-extra > gpurun_out/prof/ncu_c1.log 2>&1
for c in p2 p1; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc_attn -s 2 -c 1 -o gpurun_out/prof/$c python tools/run_config.py $c --steps 1 > gpurun_out/prof/ncu_$c.log 2>&1
done
for c in c2 c2_nested c3; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"splitk|tc_attn" -s 2 -c 2 -o gpurun_out/prof/$c python tools/run_config.py $c --steps 1 > gpurun_out/prof/ncu_$c.log 2>&1
done
echo done=$? >> gpurun_out/prof/status.txt
# C4 batch #219 (small chunk at 10K): launch list with and without the prefill key cuts
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"splitk|tc_attn|combine|append" --csv --log-file gpurun_out/prof/launches_c4_219.csv python tools/run_config.py slow --spec tools/slow_batch_c4_219.pkl --steps 2 > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"splitk|tc_attn|combine|append" --csv --log-file gpurun_out/prof/launches_c4_219_nocut.csv python tools/run_config.py slow --spec tools/slow_batch_c4_219.pkl --steps 2 --no-prefill-split > /dev/null 2>&1
