"""A/B of the host-step loop forms on one config: synchronous hg_hybrid_step_host vs
plan-ahead (hg_hybrid_step_host_async, plan the next step, synchronise), alternating
blocks of 100 steps; wall ms per step.

python tools/e2e_ahead.py c3
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch

import paper_2501_14808_b200 as hg
from paper_2501_14808_b200.harness import Workload
from synth.configs import make_config

spec = make_config(sys.argv[1] if len(sys.argv) > 1 else "c3", 0)
wl = Workload(spec)
qh, kh, vh = (x.cpu().pin_memory() for x in (wl.q, wl.k_new, wl.v_new))
oh = torch.empty(wl.out.shape, dtype=torch.bfloat16).pin_memory()
ws = torch.empty(hg.hg_hybrid_step_host_workspace_size(wl.pool, wl.batch, spec.H_q), dtype=torch.uint8, device="cuda")
st = torch.cuda.current_stream()


def sync_loop(n):
    t = time.perf_counter()
    for _ in range(n):
        hg.hg_hybrid_step_host(wl.pool, wl.batch, spec.H_q, qh, kh, vh, oh, ws)
    return (time.perf_counter() - t) / n * 1e3


def ahead_loop(n, plan=True):
    if plan:
        hg.hg_hybrid_step_host_plan(wl.pool, wl.batch, spec.H_q)
    t = time.perf_counter()
    for _ in range(n):
        hg.hg_hybrid_step_host_async(wl.pool, wl.batch, spec.H_q, qh, kh, vh, oh, ws)
        if plan:
            hg.hg_hybrid_step_host_plan(wl.pool, wl.batch, spec.H_q)
        st.synchronize()
    return (time.perf_counter() - t) / n * 1e3


def ahead_phases(n):
    hg.hg_hybrid_step_host_plan(wl.pool, wl.batch, spec.H_q)
    ta = tp = ts = 0.0
    for _ in range(n):
        a = time.perf_counter()
        hg.hg_hybrid_step_host_async(wl.pool, wl.batch, spec.H_q, qh, kh, vh, oh, ws)
        b = time.perf_counter()
        hg.hg_hybrid_step_host_plan(wl.pool, wl.batch, spec.H_q)
        c = time.perf_counter()
        st.synchronize()
        d = time.perf_counter()
        ta, tp, ts = ta + b - a, tp + c - b, ts + d - c
    return ta / n * 1e3, tp / n * 1e3, ts / n * 1e3


def plan_first(n):   # plan right before each async call: the split without the overlap
    t = time.perf_counter()
    for _ in range(n):
        hg.hg_hybrid_step_host_plan(wl.pool, wl.batch, spec.H_q)
        hg.hg_hybrid_step_host_async(wl.pool, wl.batch, spec.H_q, qh, kh, vh, oh, ws)
        st.synchronize()
    return (time.perf_counter() - t) / n * 1e3


other = hg.Batch(wl.lay.block_table, [r.c for r in spec.requests], [r.n for r in spec.requests],
                 [int(r.offline) for r in spec.requests], wl.lay.shared)


def plan_discarded(n):   # the planning work beside the GPU, but the step plans itself (other batch object)
    t = time.perf_counter()
    for _ in range(n):
        hg.hg_hybrid_step_host_async(wl.pool, other, spec.H_q, qh, kh, vh, oh, ws)
        hg.hg_hybrid_step_host_plan(wl.pool, wl.batch, spec.H_q)
        st.synchronize()
    return (time.perf_counter() - t) / n * 1e3


def sleep_between(n, plan):   # the profiled pattern: a GPU sleep after each step
    t = time.perf_counter()
    for _ in range(n):
        if plan:
            hg.hg_hybrid_step_host_plan(wl.pool, wl.batch, spec.H_q)
        hg.hg_hybrid_step_host_async(wl.pool, wl.batch, spec.H_q, qh, kh, vh, oh, ws)
        st.synchronize()
    return (time.perf_counter() - t) / n * 1e3


for _ in range(200):
    hg.hg_hybrid_step_host(wl.pool, wl.batch, spec.H_q, qh, kh, vh, oh, ws)
for rep in range(4):
    print(f"rep {rep}: sync {sync_loop(100):.3f} ms  plan-ahead {ahead_loop(100):.3f} ms  "
          f"async without plan-ahead {ahead_loop(100, plan=False):.3f} ms", flush=True)
    print("  plan-ahead phases (async call, plan, synchronise) ms: %.3f %.3f %.3f; plan right before the call %.3f ms"
          % (ahead_phases(100) + (plan_first(100),)), flush=True)
    print("  plan beside the GPU but discarded %.3f ms; plan then async (no overlap) %.3f vs async alone %.3f"
          % (plan_discarded(100), sleep_between(100, True), sleep_between(100, False)), flush=True)
