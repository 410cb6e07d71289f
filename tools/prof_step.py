"""Device timeline of one hot-path step via torch.profiler (CUPTI): kernels and
copies with their start offsets, to see where the non-kernel time goes.

python tools/prof_step.py c1            # a BASELINE config
python tools/prof_step.py c3@8          # rank 0's slice of 8-way KV-head sharding
python tools/prof_step.py c4:219        # batch #219 of the C4 sweep
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch
from torch.profiler import ProfilerActivity, profile

from paper_2501_14808_b200.harness import Workload
from synth.configs import make_config, shard_slice


def spec_of(arg):
    if arg.startswith("c4:"):
        from synth.trace import c4_batch
        return c4_batch(int(arg[3:]))
    name, _, g = arg.partition("@")
    spec = make_config(name, 0)
    return shard_slice(spec, int(g)) if g else spec


spec = spec_of(sys.argv[1] if len(sys.argv) > 1 else "c1")
wl = Workload(spec)
for _ in range(3):
    wl.step()
torch.cuda.synchronize()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    for _ in range(3):
        flush.zero_()
        torch.cuda._sleep(400000)
        wl.step()
    torch.cuda.synchronize()
evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
evs.sort(key=lambda e: e.time_range.start)
t0 = None
for e in evs:
    name = e.name[:60]
    if "sleep" in name or "fill" in name.lower() or "zero" in name.lower():
        t0 = None
        print("----", name)
        continue
    if t0 is None:
        t0 = e.time_range.start
    print("%8.1f us  +%7.1f us  %s" % (e.time_range.start - t0, e.time_range.end - e.time_range.start, name))
