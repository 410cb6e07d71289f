import sys, os; sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import time, ctypes, numpy as np, paper_2501_14808_b200 as hg
from synth.configs import make_config
from synth.layout import make_layout
spec=make_config("c3",0); lay=make_layout(spec,seed=0)
b=hg.Batch(lay.block_table,[r.c for r in spec.requests],[r.n for r in spec.requests],[int(r.offline) for r in spec.requests],lay.shared)
n=ctypes.c_int64()
o=hg.make_opts(route=1)
args=(b.ref(), spec.H_q, spec.H_kv, spec.d, lay.num_blocks, 148, 1, ctypes.byref(o))
res=[]
for rep in range(7):
    N=200; t=time.process_time()
    for i in range(N): hg.lib().hg_plan_rows(*args, None, 0, ctypes.byref(n))
    res.append((time.process_time()-t)/N*1e6)
print("min %.1f med %.1f us"%(min(res), sorted(res)[3]))
