"""tcgen05 kernel time on the prefill-heavy configs (attention only, L2 flushed,
median of 30 event-timed launches) -- the A/B harness for kernel variants:

HG_SO_OVERRIDE=paper_2501_14808_b200/var/libhygen_X.so python tools/exp_tc.py p1 p2
"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch

import paper_2501_14808_b200 as hg
from paper_2501_14808_b200.harness import Workload
from synth.configs import make_config

flush = torch.zeros(512 << 20, dtype=torch.uint8, device="cuda")


def flush_l2():
    flush[:256 << 20].zero_()
    flush[256 << 20:].view(torch.int32).amax()


tag = os.path.basename(os.environ.get("HG_SO_OVERRIDE", "default"))
for name in sys.argv[1:]:
    spec = make_config(name, 0)
    flops = sum(4 * spec.d * spec.H_q * (r.n * r.c + r.n * (r.n + 1) // 2) for r in spec.requests)
    wl = Workload(spec)
    wl.step()
    torch.cuda.synchronize()
    for mode in ("attention", "fused_step"):
        tc, step, plain = [], [], []
        for it in range(66):
            evpass = it % 2 == 0   # per-kernel events on even iterations, bare call on odd ones
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(6)] if evpass else None
            opts = hg.make_opts(events=ev)
            flush_l2()
            torch.cuda._sleep(1_000_000)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            wl.attention(opts) if mode == "attention" else wl.step(opts)
            b.record()
            torch.cuda.synchronize()
            if it >= 6:
                if evpass:
                    tc.append(ev[0].elapsed_time(ev[1]))
                else:
                    plain.append(a.elapsed_time(b))
        st = hg.hg_last_plan_stats(wl.pool)
        m, s = statistics.median(tc), statistics.median(plain)
        print(f"{tag:28s} {name} {mode:10s}: tc {m * 1e3:7.1f} us {flops / m / 1e9:7.1f} TFLOP/s (min {min(tc) * 1e3:.1f})"
              f"  call {s * 1e3:7.1f} us ({s / m:.3f}x tc)  plan {st}", flush=True)
    wl.close()
