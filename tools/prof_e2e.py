"""Device timeline of hg_hybrid_step_host (host buffers): H2D waves, kernels,
D2H, via torch.profiler (CUPTI); plus wall-clock ms per step.

python tools/prof_e2e.py c1      (HG_E2E_SERIAL=1: one input wave, for A/B)
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch
from torch.profiler import ProfilerActivity, profile

import paper_2501_14808_b200 as hg
from paper_2501_14808_b200.harness import Workload
from synth.configs import make_config

spec = make_config(sys.argv[1] if len(sys.argv) > 1 else "c1", 0)
wl = Workload(spec)
qh, kh, vh = (x.cpu().pin_memory() for x in (wl.q, wl.k_new, wl.v_new))
oh = torch.empty(wl.out.shape, dtype=torch.bfloat16).pin_memory()
ws = torch.empty(hg.hg_hybrid_step_host_workspace_size(wl.pool, wl.batch, spec.H_q), dtype=torch.uint8, device="cuda")
for _ in range(5):
    hg.hg_hybrid_step_host(wl.pool, wl.batch, spec.H_q, qh, kh, vh, oh, ws)
torch.cuda.synchronize()
n = 30
for rep in range(4):
    t0 = time.perf_counter()
    for _ in range(n):
        hg.hg_hybrid_step_host(wl.pool, wl.batch, spec.H_q, qh, kh, vh, oh, ws)
    print("wall ms/step %.3f  (HG_E2E_SERIAL=%s), loop %d" % ((time.perf_counter() - t0) / n * 1e3,
                                                            os.environ.get("HG_E2E_SERIAL"), rep))
t0 = time.perf_counter()
per = []
for _ in range(n):
    a = time.perf_counter()
    hg.hg_hybrid_step_host(wl.pool, wl.batch, spec.H_q, qh, kh, vh, oh, ws)
    per.append((time.perf_counter() - a) * 1e3)
print("per-step wall ms: " + " ".join("%.2f" % x for x in per))
t1 = time.perf_counter()
for _ in range(n):
    hg.hg_hybrid_step_host_workspace_size(wl.pool, wl.batch, spec.H_q)
print("host plan ms (workspace_size call) %.3f" % ((time.perf_counter() - t1) / n * 1e3))
# GPU time per step inside the back-to-back loop (events on the step's stream, which
# joins every other stream of the step) and the SM clock meanwhile
import threading
import pynvml
pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
clk, stop = [], [False]
def sample():
    while not stop[0]:
        clk.append(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
        time.sleep(0.002)
th = threading.Thread(target=sample)
th.start()
ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(200)]
for a, b in ev:
    a.record()
    hg.hg_hybrid_step_host(wl.pool, wl.batch, spec.H_q, qh, kh, vh, oh, ws)
    b.record()
torch.cuda.synchronize()
stop[0] = True
th.join()
g = sorted(a.elapsed_time(b) for a, b in ev)
print("loop GPU ms/step: median %.3f min %.3f max %.3f; SM MHz samples median %s min %s max %s" %
      (g[len(g) // 2], g[0], g[-1], sorted(clk)[len(clk) // 2], min(clk), max(clk)))
# same with a busy GPU between steps (diagnostic only: is it the idle clock?)
side = torch.cuda.Stream()
x = torch.empty(1 << 24, device="cuda")
for a, b in ev[:50]:
    with torch.cuda.stream(side):
        torch.cuda._sleep(1000000)
    a.record()
    hg.hg_hybrid_step_host(wl.pool, wl.batch, spec.H_q, qh, kh, vh, oh, ws)
    b.record()
torch.cuda.synchronize()
g = sorted(a.elapsed_time(b) for a, b in ev[:50])
print("loop GPU ms/step with a spinning side stream: median %.3f min %.3f" % (g[len(g) // 2], g[0]))
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    for _ in range(2):
        hg.hg_hybrid_step_host(wl.pool, wl.batch, spec.H_q, qh, kh, vh, oh, ws)
        torch.cuda._sleep(200000)
    torch.cuda.synchronize()
evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
evs.sort(key=lambda e: e.time_range.start)
t0 = None
for e in evs:
    name = e.name[:70]
    if "sleep" in name:
        t0 = None
        print("----")
        continue
    if t0 is None:
        t0 = e.time_range.start
    print("%8.1f us  +%7.1f us  %s" % (e.time_range.start - t0, e.time_range.end - e.time_range.start, name))
# back-to-back steps under the profiler (no spin between): per-step device span and copy rates
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(10):
        hg.hg_hybrid_step_host(wl.pool, wl.batch, spec.H_q, qh, kh, vh, oh, ws)
    torch.cuda.synchronize()
evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
evs.sort(key=lambda e: e.time_range.start)
steps, cur = [], []
for e in evs:
    if "Memcpy HtoD" in e.name and cur and any("DtoH" in c.name for c in cur) and \
            sum("DtoH" in c.name for c in cur) >= (2 if os.environ.get("HG_E2E_SERIAL") is None else 1):
        steps.append(cur)
        cur = []
    cur.append(e)
steps.append(cur)
for k, st in enumerate(steps):
    a, b = st[0].time_range.start, max(e.time_range.end for e in st)
    big = [e for e in st if "HtoD" in e.name and e.time_range.end - e.time_range.start > 30]
    rate = [4.2e6 / (e.time_range.end - e.time_range.start) / 1e3 for e in big]
    gap = (st[0].time_range.start - steps[k - 1][-1].time_range.end) if k else 0
    print("step %d: device span %.1f us, gap before %.1f us, big H2D GB/s %s" %
          (k, b - a, gap, ["%.0f" % r for r in rate]))
