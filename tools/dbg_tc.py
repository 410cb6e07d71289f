import sys, numpy as np, torch
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import paper_2501_14808_b200 as hg
from paper_2501_14808_b200.harness import Workload
from synth.configs import BatchSpec, Request
for Hq, Hk, ndec, grp in [(32, 4, 16, True), (32, 4, 16, False), (32, 4, 0, False), (8, 1, 0, False), (32, 32, 0, False), (64, 8, 0, False)]:
    reqs = [Request(0, 512, False)] + [Request(1024 + 37 * k, 1, True, group=(k // 2) if grp else -1, prefix_tokens=1024 if grp else 0) for k in range(ndec)]
    spec = BatchSpec("dbg", Hq, Hk, 128, 16, 0, reqs)
    wl = Workload(spec)
    for opts in [None, hg.make_opts(disable_tc=True)]:
        wl.out.fill_(float('nan'))
        wl.attention(opts)
        torch.cuda.synchronize()
        z = (wl.out[:512].float().abs().amax((1, 2)) == 0).sum().item()
        print(Hq, Hk, ndec, grp, "tc" if opts is None else "notc", "zero prefill rows", z, hg.hg_last_plan_stats(wl.pool))
