"""Device timeline (CUPTI) of two plan-ahead host steps vs two synchronous ones (C3)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch
from torch.profiler import ProfilerActivity, profile

import paper_2501_14808_b200 as hg
from paper_2501_14808_b200.harness import Workload
from synth.configs import make_config

spec = make_config(sys.argv[1] if len(sys.argv) > 1 else "c3", 0)
wl = Workload(spec)
qh, kh, vh = (x.cpu().pin_memory() for x in (wl.q, wl.k_new, wl.v_new))
oh = torch.empty(wl.out.shape, dtype=torch.bfloat16).pin_memory()
ws = torch.empty(hg.hg_hybrid_step_host_workspace_size(wl.pool, wl.batch, spec.H_q), dtype=torch.uint8, device="cuda")
st = torch.cuda.current_stream()
for _ in range(50):
    hg.hg_hybrid_step_host(wl.pool, wl.batch, spec.H_q, qh, kh, vh, oh, ws)
print("sync stats", hg.hg_last_plan_stats(wl.pool))
hg.hg_hybrid_step_host_plan(wl.pool, wl.batch, spec.H_q)
hg.hg_hybrid_step_host_async(wl.pool, wl.batch, spec.H_q, qh, kh, vh, oh, ws)
st.synchronize()
print("ahead stats", hg.hg_last_plan_stats(wl.pool))
for mode in ("sync", "ahead"):
    with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
        for _ in range(3):
            if mode == "sync":
                hg.hg_hybrid_step_host(wl.pool, wl.batch, spec.H_q, qh, kh, vh, oh, ws)
            else:
                hg.hg_hybrid_step_host_plan(wl.pool, wl.batch, spec.H_q)
                hg.hg_hybrid_step_host_async(wl.pool, wl.batch, spec.H_q, qh, kh, vh, oh, ws)
                st.synchronize()
            if os.environ.get("SLEEP"):
                torch.cuda._sleep(200000)
        torch.cuda.synchronize()
    evs = sorted([e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA],
                 key=lambda e: e.time_range.start)
    t0 = evs[0].time_range.start
    print("==", mode)
    for e in evs:
        print("%8.1f us  +%7.1f us  %s" % (e.time_range.start - t0, e.time_range.end - e.time_range.start, e.name[:60]))
    import collections
    print("host ops:")
    for e in sorted([e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CPU and "cuda" in e.name.lower()],
                    key=lambda e: e.time_range.start)[:80]:
        print("   %8.1f us  +%7.1f us  %s" % (e.time_range.start - t0, e.time_range.end - e.time_range.start, e.name[:50]))
