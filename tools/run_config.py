"""Run one synthetic config's hot-path step a few times (for ncu / quick timing).

python tools/run_config.py p2 [--steps 3] [--no-tc] [--time]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch

import paper_2501_14808_b200 as hg
from paper_2501_14808_b200.harness import Workload
from synth.configs import make_config

ap = argparse.ArgumentParser()
ap.add_argument("config")
ap.add_argument("--steps", type=int, default=3)
ap.add_argument("--no-tc", action="store_true")
ap.add_argument("--no-prefix", action="store_true")
ap.add_argument("--time", action="store_true")
ap.add_argument("--split", type=int, default=0)
ap.add_argument("--no-prefill-split", action="store_true")
ap.add_argument("--spec", default=None, help="pickled BatchSpec instead of a named config")
a = ap.parse_args()
if a.spec:
    import pickle
    spec = pickle.load(open(a.spec, "rb"))
else:
    spec = make_config(a.config, 0)
wl = Workload(spec)
opts = hg.make_opts(disable_tc=a.no_tc, disable_prefix_pass=a.no_prefix, split_tokens=a.split,
                    disable_prefill_split=a.no_prefill_split)
for _ in range(2):
    wl.step(opts)
torch.cuda.synchronize()
ev = [[torch.cuda.Event(enable_timing=True) for _ in range(6)] for _ in range(a.steps)]
ops = [hg.make_opts(disable_tc=a.no_tc, disable_prefix_pass=a.no_prefix, split_tokens=a.split, events=e,
                   disable_prefill_split=a.no_prefill_split) for e in ev]
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
tot = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(a.steps)]
for k in range(a.steps):
    flush.zero_()
    if os.environ.get("HG_HOST_AHEAD"):
        torch.cuda._sleep(400000)   # keep the GPU busy so the host enqueues the step ahead of it
    tot[k][0].record()
    wl.step(ops[k])
    tot[k][1].record()
torch.cuda.synchronize()
if a.time:
    st = hg.hg_last_plan_stats(wl.pool)
    for k in range(a.steps):
        e = ev[k]
        lead = tot[k][0].elapsed_time(e[2]) if st["splitk_items"] else 0.0
        lead_tc = tot[k][0].elapsed_time(e[0]) if st["tc_tiles"] else 0.0
        print("   lead to tc start %.4f" % lead_tc)
        tail = e[3].elapsed_time(tot[k][1]) if st["splitk_items"] else 0.0
        print(a.config, "split", a.split, "step %.4f lead %.4f tail %.4f" % (tot[k][0].elapsed_time(tot[k][1]), lead, tail), "tc %.4f" % (e[0].elapsed_time(e[1]) if st["tc_tiles"] else 0),
              "splitk %.4f" % (e[2].elapsed_time(e[3]) if st["splitk_items"] else 0),
              "comb %.4f" % (e[4].elapsed_time(e[5]) if st["combine_rows"] else 0), st)
