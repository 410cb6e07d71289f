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
n = int(st["splitk_items"])   # CTAs (the SM ids follow the start / end pairs)
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
if os.environ.get("HG_TRACE_TAIL"):
    # CTA b runs LPT item b (one item per CTA): who ends last, and how long the
    # first wave's items take as a function of their LPT rank
    order = np.argsort(e)[::-1][:24]
    print("last-ending CTAs: lpt_rank start end dur")
    for b in order:
        print(f"  {b:5d} {s[b]:7.1f} {e[b]:7.1f} {e[b] - s[b]:6.1f}")
    for lo, hi in [(0, 50), (50, 150), (150, 300), (300, 444), (444, 600), (600, n - 40), (n - 40, n)]:
        if hi > lo:
            d = e[lo:hi] - s[lo:hi]
            print(f"  rank [{lo},{hi}): start {np.median(s[lo:hi]):6.1f} end med {np.median(e[lo:hi]):6.1f} "
                  f"max {e[lo:hi].max():6.1f} dur med {np.median(d):6.1f} min {d.min():6.1f} max {d.max():6.1f}")
    # SM of each CTA (written after the start / end pairs): do the slow first-wave CTAs
    # share SMs (or GPCs)?
    sm = t[2 * n:3 * n].astype(np.int64)
    d = e - s
    first = np.arange(n) < min(444, n)
    big = first & (np.arange(n) < 300)
    if big.any():
        db = d[big]
        slow = big & (d > np.percentile(db, 90))
        fast = big & (d < np.percentile(db, 10))
        print("  slowest 10% of ranks [0,300): SMs", sorted(sm[slow].tolist()))
        print("  fastest 10% of ranks [0,300): SMs", sorted(sm[fast].tolist()))
        per_sm = {}
        for b in np.flatnonzero(big):
            per_sm.setdefault(int(sm[b]), []).append(d[b])
        avg = np.array([np.mean(per_sm.get(k, [np.nan])) for k in range(148)])
        print("  mean big-item duration by SM id (rows of 16 SMs):")
        for r0 in range(0, 148, 16):
            print("   " + " ".join(f"{x:5.1f}" for x in avg[r0:r0 + 16]))
