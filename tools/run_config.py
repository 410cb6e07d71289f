"""Run a few fused steps of one config (optionally a shard slice) for ncu captures.

python tools/run_config.py c3@8 [--no-tc] [--steps N]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch

import paper_2501_14808_b200 as hg
from paper_2501_14808_b200.harness import Workload
from synth.configs import make_config, shard_slice

ap = argparse.ArgumentParser()
ap.add_argument("config")
ap.add_argument("--no-tc", action="store_true")
ap.add_argument("--route", type=int, default=0)
ap.add_argument("--steps", type=int, default=3)
a = ap.parse_args()
name, _, g = a.config.partition("@")
spec = make_config(name, 0)
spec = shard_slice(spec, int(g)) if g else spec
wl = Workload(spec)
opts = hg.make_opts(disable_tc=a.no_tc, route=a.route)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for _ in range(a.steps):
    flush.zero_()
    wl.step(opts)
torch.cuda.synchronize()
print(hg.hg_last_plan_stats(wl.pool))
