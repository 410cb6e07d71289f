"""SM clock / power / throttle reasons while one config's step runs back to back
for ~2 s (NVML, 1 ms period): is a kernel clock- (power-) limited?

python tools/clock_probe.py p2 [seconds]
"""
import os
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import pynvml
import torch

from paper_2501_14808_b200.harness import Workload
from synth.configs import make_config

name = sys.argv[1] if len(sys.argv) > 1 else "p2"
secs = float(sys.argv[2]) if len(sys.argv) > 2 else 2.0
spec = make_config(name, 0)
wl = Workload(spec)
for _ in range(3):
    wl.step()
torch.cuda.synchronize()
pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
samples, stop = [], [False]


def run():
    while not stop[0]:
        samples.append((pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                        pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0,
                        pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)))
        time.sleep(0.001)


th = threading.Thread(target=run)
th.start()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
n = 0
t0 = time.perf_counter()
e0.record()
while time.perf_counter() - t0 < secs:
    for _ in range(20):
        wl.step()
    n += 20
    torch.cuda.synchronize()
e1.record()
torch.cuda.synchronize()
stop[0] = True
th.join()
ms = e0.elapsed_time(e1) / n
s = sorted(x[0] for x in samples[len(samples) // 4:])
p = sorted(x[1] for x in samples[len(samples) // 4:])
reasons = 0
for x in samples:
    reasons |= x[2]
print("%s: %d steps, %.4f ms/step back to back; SM MHz (last 3/4) median %d min %d max %d; "
      "power W median %.0f max %.0f; reasons mask 0x%x" %
      (name, n, ms, s[len(s) // 2], s[0], s[-1], p[len(p) // 2], p[-1], reasons))
