"""Per-rank cost of the sharded step on one GPU: rank 0's KV-head slice of a config at
G = 1/2/4/8 through (a) hg_hybrid_step (no communicator), (b) hg_hybrid_step_tp on a
1-rank peer window (entry barrier, window stores, exit barrier), device time, L2
flushed, GPU kept busy while the host plans; median of 40.

python tools/exp_tp.py c3 [c1]
"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch

import paper_2501_14808_b200 as hg
from paper_2501_14808_b200.harness import Workload
from synth.configs import make_config, shard_slice

flush = torch.zeros(512 << 20, dtype=torch.uint8, device="cuda")


def flush_l2():
    flush[:256 << 20].zero_()
    flush[256 << 20:].view(torch.int32).amax()


def timed(fn, reps=40):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        flush_l2()
        torch.cuda._sleep(1_000_000)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    return statistics.median(ts)


tag = os.environ.get("EXP_TAG", "")
for name in sys.argv[1:]:
    spec = make_config(name, 0)
    base = None
    for G in (1, 2, 4, 8):
        local = shard_slice(spec, G)
        wl = Workload(local)
        comm = hg.Comm(None, 0, 1, torch.cuda.current_device())
        h = comm.hg_comm_window_create(local.T * local.H_q * local.d * 2)
        comm.hg_comm_window_open([h])
        win = comm.window((local.T, local.H_q, local.d))
        ws = torch.empty(hg.hg_hybrid_attention_tp_workspace_size(wl.pool, comm, wl.batch, local.H_q),
                         dtype=torch.uint8, device="cuda")
        t_fused = timed(lambda: wl.step())
        t_tp = timed(lambda: hg.hg_hybrid_step_tp(wl.pool, comm, wl.batch, local.H_q, wl.q, wl.k_new, wl.v_new, win, ws))
        st = hg.hg_last_plan_stats(wl.pool)
        base = t_tp if G == 1 else base
        print(f"{tag}{name}@{G}: fused step {t_fused:7.1f} us  tp step {t_tp:7.1f} us  (x{base / t_tp:.2f} vs G=1)  "
              f"plan {st}", flush=True)
        comm.close()
        wl.close()
