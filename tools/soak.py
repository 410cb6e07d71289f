"""Soak test of the long-lived state (descriptor / staging rings, peer-window epochs, the
folded barriers' tickets, plan-ahead slots): many back-to-back steps, output checked
against the first step's bits every `every` steps.

python tools/soak.py [steps]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch

import paper_2501_14808_b200 as hg
from paper_2501_14808_b200.harness import Workload
from synth.configs import make_config, shard_slice

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
every = 997

# 1) the sharded HBM step (C3's 8-way slice) on a 1-rank peer window
local = shard_slice(make_config("c3", 0), 8)
wl = Workload(local)
comm = hg.Comm(None, 0, 1, torch.cuda.current_device())
comm.hg_comm_window_open([comm.hg_comm_window_create(local.T * local.H_q * local.d * 2)])
win = comm.window((local.T, local.H_q, local.d))
ws = torch.empty(hg.hg_hybrid_attention_tp_workspace_size(wl.pool, comm, wl.batch, local.H_q),
                 dtype=torch.uint8, device="cuda")
hg.hg_hybrid_step_tp(wl.pool, comm, wl.batch, local.H_q, wl.q, wl.k_new, wl.v_new, win, ws)
torch.cuda.synchronize()
ref = win.clone()
t0 = time.perf_counter()
bad = 0
for k in range(steps):
    hg.hg_hybrid_step_tp(wl.pool, comm, wl.batch, local.H_q, wl.q, wl.k_new, wl.v_new, win, ws)
    if k % every == 0:
        torch.cuda.synchronize()
        bad += int(not torch.equal(win.view(torch.int16), ref.view(torch.int16)))
torch.cuda.synchronize()
bad += int(not torch.equal(win.view(torch.int16), ref.view(torch.int16)))
print(f"sharded step (c3@8, 1-rank window): {steps} steps in {time.perf_counter() - t0:.2f} s, "
      f"{bad} mismatching checks, plan {hg.hg_last_plan_stats(wl.pool)}", flush=True)
comm.close()
wl.close()

# 2) the host step, plan-ahead loop (C3)
spec = make_config("c3", 0)
wl = Workload(spec)
qh, kh, vh = (x.cpu().pin_memory() for x in (wl.q, wl.k_new, wl.v_new))
oh = torch.empty(wl.out.shape, dtype=torch.bfloat16).pin_memory()
ws = torch.empty(hg.hg_hybrid_step_host_workspace_size(wl.pool, wl.batch, spec.H_q), dtype=torch.uint8, device="cuda")
hg.hg_hybrid_step_host(wl.pool, wl.batch, spec.H_q, qh, kh, vh, oh, ws)
ref = oh.clone()
st = torch.cuda.current_stream()
n2 = steps // 4
t0 = time.perf_counter()
bad = 0
hg.hg_hybrid_step_host_plan(wl.pool, wl.batch, spec.H_q)
for k in range(n2):
    hg.hg_hybrid_step_host_async(wl.pool, wl.batch, spec.H_q, qh, kh, vh, oh, ws)
    hg.hg_hybrid_step_host_plan(wl.pool, wl.batch, spec.H_q)
    st.synchronize()
    if k % every == 0:
        bad += int(not torch.equal(oh.view(torch.int16), ref.view(torch.int16)))
bad += int(not torch.equal(oh.view(torch.int16), ref.view(torch.int16)))
print(f"host step plan-ahead (c3): {n2} steps in {time.perf_counter() - t0:.2f} s, {bad} mismatching checks",
      flush=True)
