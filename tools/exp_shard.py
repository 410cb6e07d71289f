"""A/B of plan switches on one rank's slice of KV-head sharding (device time of
the fused step, L2 flushed, GPU kept busy while the host plans), plus the
per-kernel split from the library's events.

python tools/exp_shard.py c3@8 c3@4 c3 c1@8
"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch

import paper_2501_14808_b200 as hg
from paper_2501_14808_b200.harness import Workload
from synth.configs import make_config, shard_slice


def spec_of(arg):
    name, _, g = arg.partition("@")
    spec = make_config(name, 0)
    return shard_slice(spec, int(g)) if g else spec


VARIANTS = {"default": {}, "tc_route": dict(route=1), "hbm_route": dict(route=2), "no_tc": dict(disable_tc=True), "no_prefix": dict(disable_prefix_pass=True),
            }
if os.environ.get("EXP_VARIANTS"):
    VARIANTS = {k: v for k, v in VARIANTS.items() if k in os.environ["EXP_VARIANTS"].split(",")}
flush = torch.zeros(512 << 20, dtype=torch.uint8, device="cuda")
def flush_l2():   # write 256 MB, then read another 256 MB: L2 ends full of clean, unrelated lines
    flush[:256 << 20].zero_()
    flush[256 << 20:].view(torch.int32).amax()

for arg in sys.argv[1:]:
    spec = spec_of(arg)
    wl = Workload(spec)
    for vname, kw in VARIANTS.items():
        for _ in range(3):
            wl.step(hg.make_opts(**kw))
        torch.cuda.synchronize()
        ts, ks = [], []
        for ev_pass in (False, True):
            for _ in range(30):
                ev = [torch.cuda.Event(enable_timing=True) for _ in range(6)] if ev_pass else None
                opts = hg.make_opts(events=ev, **kw)   # (records the events once: outside the timed region)
                flush_l2()
                torch.cuda._sleep(1_000_000)
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                wl.step(opts)
                b.record()
                torch.cuda.synchronize()
                st = hg.hg_last_plan_stats(wl.pool)
                if not ev_pass:   # step time without per-kernel events (PDL pairs intact)
                    ts.append(a.elapsed_time(b))
                    continue
                k = {"step_ev": a.elapsed_time(b)}
                if st["tc_tiles"]:
                    k["tc"] = ev[0].elapsed_time(ev[1])
                    k["tc_start"] = a.elapsed_time(ev[0])
                if st["splitk_items"]:
                    k["sk"] = ev[2].elapsed_time(ev[3])
                    k["sk_start"] = a.elapsed_time(ev[2])
                if st["combine_rows"]:
                    k["comb"] = ev[4].elapsed_time(ev[5])
                ks.append(k)
        med = statistics.median(ts)
        kk = {n: statistics.median(x[n] for x in ks if n in x) for n in ks[0]}
        print(f"{arg:8s} {vname:10s} step {med*1e3:7.1f} us  " +
              "  ".join(f"{n} {v*1e3:6.1f}" for n, v in kk.items()) + f"  plan {st}", flush=True)
    wl.close()
