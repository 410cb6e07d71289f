"""Timeline of the exp_shard-style timed loop (timing events + per-kernel events)
under the profiler, plus the host time of each step() call."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch
from torch.profiler import ProfilerActivity, profile

import paper_2501_14808_b200 as hg
from paper_2501_14808_b200.harness import Workload
from synth.configs import make_config, shard_slice

name, _, g = sys.argv[1].partition("@")
spec = make_config(name, 0)
spec = shard_slice(spec, int(g)) if g else spec
use_ev = len(sys.argv) > 2 and sys.argv[2] == "ev"
wl = Workload(spec)
for _ in range(3):
    wl.step()
torch.cuda.synchronize()
flush = torch.zeros(512 << 20, dtype=torch.uint8, device="cuda")
def flush_l2():   # write 256 MB, then read another 256 MB: L2 ends full of clean, unrelated lines
    flush[:256 << 20].zero_()
    flush[256 << 20:].view(torch.int32).amax()

host = []
with profile(activities=[ProfilerActivity.CUDA], acc_events=True) as prof:
    for _ in range(4):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(6)]
        flush_l2()
        torch.cuda._sleep(1_000_000)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        h0 = time.perf_counter()
        wl.step(hg.make_opts(events=ev) if use_ev else None)
        host.append((time.perf_counter() - h0) * 1e6)
        b.record()
        torch.cuda.synchronize()
        print("step event ms", a.elapsed_time(b), "host us", host[-1])
evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
evs.sort(key=lambda e: e.time_range.start)
t0 = None
for e in evs:
    n = e.name[:60]
    if "spin" in n:
        t0 = e.time_range.end
        print("---- spin end")
        continue
    if t0 is None:
        continue
    print("%8.1f us  +%7.1f us  %s" % (e.time_range.start - t0, e.time_range.end - e.time_range.start, n))
