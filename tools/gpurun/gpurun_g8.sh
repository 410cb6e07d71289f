mkdir -p gpurun_out/g8e
for w in 1 2 3 4; do
HG_SK_WAVES=$w HG_HOST_AHEAD=1 timeout 300 python tools/run_config.py x --spec tools/c1_shard_g8.pkl --time --steps 10 2>&1 | grep "step" | tail -6 > gpurun_out/g8e/g8_w$w.log
done
python - <<'PY'
import pickle
from synth.configs import make_config
for G in (2, 4):
    s = make_config("c1", 0)
    pickle.dump(s.with_(H_kv=32 // G, H_q=32 // G), open(f"gpurun_out/g8e/c1_g{G}.pkl", "wb"))
PY
for G in 2 4; do for w in 1 2; do
HG_SK_WAVES=$w HG_HOST_AHEAD=1 timeout 300 python tools/run_config.py x --spec gpurun_out/g8e/c1_g$G.pkl --time --steps 10 2>&1 | grep "step" | tail -6 > gpurun_out/g8e/g${G}_w$w.log
done; done
