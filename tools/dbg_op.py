import sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_2501_14808_b200 as hg
from paper_2501_14808_b200.harness import Workload
from synth.configs import make_config
spec = make_config("c3", 0)
spec = spec.with_(requests=spec.requests[:1] + spec.requests[1:257:16])
wl = Workload(spec)
world, rank = 2, int(sys.argv[1]) if len(sys.argv) > 1 else 0
Hk, Hq, d = spec.H_kv // world, spec.H_q // world, spec.d
kc = wl.k_cache[:, rank*Hk:(rank+1)*Hk].contiguous(); vc = wl.v_cache[:, rank*Hk:(rank+1)*Hk].contiguous(); ql = wl.q[:, rank*Hq:(rank+1)*Hq].contiguous()
pool = hg.KVPool(kc, vc, wl.lay.num_blocks, spec.B, Hk, d, 0)
o = torch.full((spec.T, Hq, d), float('nan'), dtype=torch.bfloat16, device='cuda')
ws = torch.empty(hg.hg_hybrid_attention_workspace_size(pool, wl.batch, Hq) + (1 << 20), dtype=torch.uint8, device='cuda')
hg.hg_hybrid_attention(pool, wl.batch, Hq, ql, o, None, ws)
torch.cuda.synchronize()
print("T", spec.T, "nan rows", torch.isnan(o.float()).any(-1).any(-1).nonzero().flatten()[:20].tolist(), hg.hg_last_plan_stats(pool))
comm = hg.Comm(None, 0, 1, 0)
from synth.values import KIND_W, matrix
W = matrix(11, KIND_W, 0, Hq * d, 512, scale=0.01, device='cuda')
y = torch.full((spec.T, 512), float('nan'), dtype=torch.bfloat16, device='cuda')
ws3 = torch.empty(hg.hg_hybrid_attention_tp_proj_workspace_size(pool, comm, wl.batch, Hq), dtype=torch.uint8, device='cuda')
hg.hg_hybrid_attention_tp_proj(pool, comm, wl.batch, Hq, ql, W, 512, y, ws3)
torch.cuda.synchronize()
print("y nan rows", torch.isnan(y.float()).any(-1).nonzero().flatten()[:20].tolist())
ref = o.reshape(spec.T, -1).double().cpu() @ W.double().cpu()
print("rel", ((y.double().cpu() - ref).norm() / ref.norm()).item())
print("o[:264] absmax", o[:264].float().abs().max().item(), "o[264:] absmax", o[264:].float().abs().max().item())
print("q[:264] absmax", ql[:264].float().abs().max().item())
print("zero rows", (o.float().abs().amax((1, 2)) == 0).nonzero().flatten()[:10].tolist(), (o.float().abs().amax((1, 2)) == 0).sum().item())
