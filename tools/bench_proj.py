"""Time hg_out_proj_rs on one GPU (G = 1: the GEMM with its epilogue stores).

python tools/bench_proj.py [T K N ...]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2501_14808_b200 as hg
from synth.values import KIND_O, KIND_W, matrix

shapes = [(768, 8192, 8192), (768, 1024, 8192), (576, 4096, 4096), (4096, 4096, 4096), (8192, 8192, 8192)]
if len(sys.argv) > 3:
    a = list(map(int, sys.argv[1:]))
    shapes = [tuple(a[i:i + 3]) for i in range(0, len(a), 3)]
comm = hg.Comm(None, 0, 1, torch.cuda.current_device())
for T, K, N in shapes:
    O = matrix(1, KIND_O, 0, T, K, device="cuda")
    W = matrix(1, KIND_W, 0, K, N, scale=K ** -0.5, device="cuda")
    y = torch.empty((T, N), dtype=torch.bfloat16, device="cuda")
    for _ in range(3):
        hg.hg_out_proj_rs(comm, T, K, N, O, W, y)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 20
    s.record()
    for _ in range(reps):
        hg.hg_out_proj_rs(comm, T, K, N, O, W, y)
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / reps
    ref = torch.matmul(O, W)
    torch.cuda.synchronize()
    s.record()
    for _ in range(reps):
        torch.matmul(O, W, out=ref)
    e.record()
    torch.cuda.synchronize()
    ms_cublas = s.elapsed_time(e) / reps
    fl = 2.0 * T * K * N
    print(f"T {T} K {K} N {N}: {ms * 1e3:.1f} us  {fl / ms / 1e9:.0f} TFLOP/s   (cuBLAS {ms_cublas * 1e3:.1f} us, "
          f"{fl / ms_cublas / 1e9:.0f} TFLOP/s)  max|diff| {float((y.float() - ref.float()).abs().max()):.3g}")
comm.close()
