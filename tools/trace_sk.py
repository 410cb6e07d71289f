"""Split-K grid occupancy over time: every CTA's %globaltimer start / end
(hg_attn_opts.debug_sk_trace), for one config or shard slice.

python tools/trace_sk.py c3@8 [route]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

import paper_2501_14808_b200 as hg
from paper_2501_14808_b200.harness import Workload
from synth.configs import make_config, shard_slice

name, _, g = sys.argv[1].partition("@")
route = int(sys.argv[2]) if len(sys.argv) > 2 else 0
spec = make_config(name, 0)
spec = shard_slice(spec, int(g)) if g else spec
wl = Workload(spec)
flush = torch.zeros(512 << 20, dtype=torch.uint8, device="cuda")
tr = torch.zeros(1 << 20, dtype=torch.int64, device="cuda")
for rep in range(4):
    flush[:256 << 20].zero_()
    flush[256 << 20:].view(torch.int32).amax()
    tr.zero_()
    o = hg.make_opts(route=route)
    o.debug_sk_trace = tr.data_ptr()
    wl.step(o)
    torch.cuda.synchronize()
st = hg.hg_last_plan_stats(wl.pool)
t = tr.cpu().numpy()
n = int((t != 0).sum() // 2)
s, e = t[0:2 * n:2], t[1:2 * n:2]
t0 = s.min()
s, e = (s - t0) / 1e3, (e - t0) / 1e3
print(f"{sys.argv[1]}: {n} split-K CTAs, first start 0, last start {s.max():.1f} us, last end {e.max():.1f} us, "
      f"CTA duration median {np.median(e - s):.1f} us (min {np.min(e - s):.1f}, max {np.max(e - s):.1f}); plan {st}")
edges = np.arange(0, e.max() + 2, 2.0)
active = [int(((s <= x) & (e > x)).sum()) for x in edges]
print("time(us) active CTAs")
for x, a in zip(edges, active):
    print(f"{x:7.1f} {a:5d} " + "#" * (a // 8))
