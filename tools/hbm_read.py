import torch
x = torch.empty(4 << 30, dtype=torch.uint8, device="cuda")   # 4 GB
x.fill_(1)
xf = x.view(torch.float32)
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
best = 1e9
for _ in range(10):
    torch.cuda.synchronize(); s.record(); r = xf.sum(); e.record(); torch.cuda.synchronize()
    best = min(best, s.elapsed_time(e))
print("torch sum read: %.1f GB/s" % (x.numel() / best / 1e6))
# max read with a simple vectorized kernel via torch: amax over int64 view
xi = x.view(torch.int64)
best = 1e9
for _ in range(10):
    torch.cuda.synchronize(); s.record(); r = xi.amax(); e.record(); torch.cuda.synchronize()
    best = min(best, s.elapsed_time(e))
print("torch amax read: %.1f GB/s" % (x.numel() / best / 1e6))
y = torch.empty_like(x)
best = 1e9
for _ in range(10):
    torch.cuda.synchronize(); s.record(); y.copy_(x); e.record(); torch.cuda.synchronize()
    best = min(best, s.elapsed_time(e))
print("copy (r+w): %.1f GB/s" % (2 * x.numel() / best / 1e6))
