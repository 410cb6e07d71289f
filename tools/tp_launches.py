"""The sharded serving step's kernels, for an ncu launch list: rank 0's KV-head slice
of a config at G ranks through hg_hybrid_step_tp on a 1-rank peer window, `steps`
calls (run under `ncu --metrics gpu__time_duration.sum --csv`; every launch of the
library's kernels in these calls is one line).

python tools/tp_launches.py c3 8 [steps]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch

import paper_2501_14808_b200 as hg
from paper_2501_14808_b200.harness import Workload
from synth.configs import make_config, shard_slice

name, G = sys.argv[1], int(sys.argv[2])
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
local = shard_slice(make_config(name, 0), G)
wl = Workload(local)
comm = hg.Comm(None, 0, 1, torch.cuda.current_device())
comm.hg_comm_window_open([comm.hg_comm_window_create(local.T * local.H_q * local.d * 2)])
win = comm.window((local.T, local.H_q, local.d))
ws = torch.empty(hg.hg_hybrid_attention_tp_workspace_size(wl.pool, comm, wl.batch, local.H_q),
                 dtype=torch.uint8, device="cuda")
torch.cuda.synchronize()
for _ in range(steps):
    hg.hg_hybrid_step_tp(wl.pool, comm, wl.batch, local.H_q, wl.q, wl.k_new, wl.v_new, win, ws)
torch.cuda.synchronize()
print(f"{name}@{G}: {steps} sharded steps, plan {hg.hg_last_plan_stats(wl.pool)}")
comm.close()
wl.close()
