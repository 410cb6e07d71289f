"""tcgen05 grid balance: every CTA's start / end (%globaltimer, debug_trace) for the
attention of a prefill-heavy config, L2 flushed; median over reps of the makespan
and the spread of CTA end times (the planner's assign_tc decides it).

python tools/trace_tc_grid.py p1 p2
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

import paper_2501_14808_b200 as hg
from paper_2501_14808_b200.harness import Workload
from synth.configs import make_config

tag = os.path.basename(os.environ.get("HG_SO_OVERRIDE", "default"))
flush = torch.zeros(512 << 20, dtype=torch.uint8, device="cuda")
for name in sys.argv[1:]:
    wl = Workload(make_config(name, 0))
    wl.step()
    tr = torch.zeros(8192, dtype=torch.int64, device="cuda")
    mks, ends = [], []
    for rep in range(12):
        flush[:256 << 20].zero_()
        flush[256 << 20:].view(torch.int32).amax()
        tr.zero_()
        o = hg.make_opts()
        o.debug_trace = tr.data_ptr()
        wl.attention(o)
        torch.cuda.synchronize()
        c = tr.cpu().numpy()[4096:4096 + 4 * 148].reshape(-1, 4)
        c = c[c[:, 3] > 0]
        ns0 = c[:, 2].min()
        e = np.sort((c[:, 3] - ns0) / 1e3)
        if rep >= 2:
            mks.append(e[-1])
            ends.append(e)
    st = hg.hg_last_plan_stats(wl.pool)
    e = np.median(np.array(ends), axis=0)
    print(f"{tag} {name}: makespan median {np.median(mks):.1f} us (min {min(mks):.1f}); CTA end p10 {e[int(.1 * len(e))]:.1f} "
          f"p50 {e[len(e) // 2]:.1f} p90 {e[int(.9 * len(e))]:.1f} max {e[-1]:.1f}; tiles {st['tc_tiles']}")
    wl.close()
