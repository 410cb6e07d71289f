"""Timeline of tcgen05 CTA 0 (debug_trace): where does a KV tile's time go?"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2501_14808_b200 as hg
from paper_2501_14808_b200.harness import Workload
from synth.configs import make_config
spec = make_config(sys.argv[1] if len(sys.argv) > 1 else "p2", 0)
wl = Workload(spec)
wl.step()
tr = torch.zeros(8192, dtype=torch.int64, device="cuda")
o = hg.make_opts()
o.debug_trace = tr.data_ptr()
wl.attention(o)
torch.cuda.synchronize()
t = tr.cpu().numpy()
base = t[t > 0].min()
t = np.where(t > 0, t - base, -1)
print("j | TMA-issue | PFULL0 seen  PV0+QK0 issued | PFULL1 seen  PV1+QK1 issued | S0 ready P0 done | S1 ready P1 done")
for j in range(0, 40):
    print(j, t[1024 + 2 * j], "|", t[8 * j], t[8 * j + 1], "|", t[8 * j + 2], t[8 * j + 3], "|",
          t[512 + 2 * j], t[512 + 2 * j + 1], "|", t[768 + 2 * j], t[768 + 2 * j + 1])

print("softmax tile 0: S ready -> S loaded -> max/bump done -> first half exps done -> PHALF arrived -> P done")
for j in range(0, 20):
    a = [t[512 + 2 * j]] + [t[2048 + 8 * j + k] for k in range(4)] + [t[512 + 2 * j + 1]]
    print(j, a, "deltas", [a[k + 1] - a[k] for k in range(5)])

# per-CTA start / end (clock64, %globaltimer ns) of the whole grid
c = tr.cpu().numpy()[4096:4096 + 4 * 148].reshape(-1, 4)
c = c[c[:, 1] > 0]
ns0 = c[:, 2].min()
busy_ns = c[:, 3] - c[:, 2]
mhz = (c[:, 1] - c[:, 0]) / np.maximum(busy_ns, 1) * 1e3
print(f"grid: {len(c)} CTAs, makespan {(c[:, 3].max() - ns0) / 1e3:.1f} us, CTA busy min/median/max "
      f"{busy_ns.min() / 1e3:.1f} / {np.median(busy_ns) / 1e3:.1f} / {busy_ns.max() / 1e3:.1f} us, "
      f"start skew {(c[:, 2].max() - ns0) / 1e3:.1f} us, SM clock {np.median(mhz):.0f} MHz (min {mhz.min():.0f})")
