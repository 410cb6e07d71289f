"""Counter-based token values: identical bf16 bits on CPU and CUDA.

value(seed, kind, cid, pos, head, dim) is a pure function of integer
coordinates.  It is built from 32-bit integer mixing (murmur3 ``fmix32``)
evaluated in int64 torch tensors (exact, wrap-around products masked to 32
bits), followed by an Irwin-Hall sum of four 24-bit uniforms, one int->fp32
conversion (round-to-nearest-even), one fp32 multiply by a constant and one
fp32->bf16 round-to-nearest-even.  Every step is exactly specified by IEEE-754
and two's-complement arithmetic, so torch-CPU and torch-CUDA give the same
bits (checked by tests/test_synth.py on CPU and tests/test_gpu_parity.py on
GPU).

The distribution has mean 0 and variance 1 (sum of four U[0,1) has variance
1/3, rescaled by sqrt(3)), i.e. the "N(0,1)-scale" activations of DESIGN.md
§Inputs; ``q_scale`` multiplies Q before rounding for the "peaked" variants.

Content ids decouple *what* a token holds from *where* it is stored: a shared
prefix has one content id per group no matter whether its blocks are
physically shared or privately copied.
"""
from __future__ import annotations

import math

import torch

M32 = 0xFFFFFFFF
KIND_Q, KIND_K, KIND_V = 0, 1, 2
_SCALE = math.sqrt(3.0) / float(1 << 24)
GROUP_CID_BASE = 1 << 20


def _fmix32_int(h: int) -> int:
    h &= M32
    h ^= h >> 16
    h = (h * 0x85EBCA6B) & M32
    h ^= h >> 13
    h = (h * 0xC2B2AE35) & M32
    h ^= h >> 16
    return h


def _fmix32(h: torch.Tensor) -> torch.Tensor:
    h = h ^ (h >> 16)
    h = (h * 0x85EBCA6B) & M32
    h = h ^ (h >> 13)
    h = (h * 0xC2B2AE35) & M32
    h = h ^ (h >> 16)
    return h


def gen_block(seed: int, kind: int, cid: int, pos: torch.Tensor, heads: int, dim: int,
              scale: float = 1.0, device=None) -> torch.Tensor:
    """bf16 tensor [len(pos)][heads][dim] for content id ``cid`` at positions ``pos``."""
    device = device if device is not None else pos.device
    base = _fmix32_int(_fmix32_int(seed * 0x9E3779B1 + kind * 0x632BE5AB) ^ (cid & M32))
    p = pos.to(device=device, dtype=torch.int64).reshape(-1, 1, 1)
    hd = (torch.arange(heads, device=device, dtype=torch.int64).reshape(1, -1, 1) * dim
          + torch.arange(dim, device=device, dtype=torch.int64).reshape(1, 1, -1))
    h = _fmix32((p * 0x27D4EB2F + base) & M32)
    h = _fmix32(h ^ hd)
    s = torch.zeros_like(h)
    for k in range(4):
        s = s + (_fmix32(h ^ ((k + 1) * 0x9E3779B9 & M32)) >> 8)
    x = (s - (1 << 25)).to(torch.float32) * torch.tensor(_SCALE, dtype=torch.float32, device=device)
    if scale != 1.0:
        x = x * torch.tensor(scale, dtype=torch.float32, device=device)
    return x.to(torch.bfloat16)


def segments(spec, i: int):
    """[(start, end, content id)] covering request i's positions: its prefix
    groups root to leaf (nested sharing, NEXT-3), then its own content."""
    r = spec.requests[i]
    out = []
    if r.group >= 0 and r.prefix_tokens > 0:
        chain = spec.group_chain(r.group)
        for k, (g, start) in enumerate(chain):
            end = chain[k + 1][1] if k + 1 < len(chain) else r.prefix_tokens
            if end > start:
                out.append((start, end, GROUP_CID_BASE + g))
    out.append((r.prefix_tokens if r.group >= 0 else 0, 1 << 62, own_cid(spec, i)))
    return out


def content_id(spec, i: int, pos: int) -> int:
    """Content id of request i's token at absolute position ``pos``."""
    for a, b, cid in segments(spec, i):
        if a <= pos < b:
            return cid
    raise ValueError(pos)


def own_cid(spec, i: int) -> int:
    r = spec.requests[i]
    return i if r.cid < 0 else r.cid


def kv_values(spec, i: int, start: int, end: int, kind: int, device="cpu") -> torch.Tensor:
    """K (kind=KIND_K) or V (kind=KIND_V) rows of request i for positions [start, end).

    Returns bf16 [end-start][H_kv][d]; positions inside the group prefix take
    the content of the group owning them (root to leaf), the rest the request's
    own content.
    """
    parts = []
    for a, b, cid in segments(spec, i):
        lo, hi = max(start, a), min(end, b)
        if lo < hi:
            pos = torch.arange(lo, hi, dtype=torch.int64)
            parts.append(gen_block(spec.seed, kind, cid, pos, spec.H_kv, spec.d, device=device))
    if not parts:
        return torch.empty((0, spec.H_kv, spec.d), dtype=torch.bfloat16, device=device)
    return torch.cat(parts, 0) if len(parts) > 1 else parts[0]


def q_values(spec, device="cpu", requests=None) -> torch.Tensor:
    """Q of the batch's new tokens, bf16 [T][H_q][d], rows in request order.

    Request i's row j carries the query of absolute position c_i + j, so the
    same logical token has the same query however the prompt is chunked.
    ``requests`` optionally restricts to a subset (rows concatenated in that order).
    """
    idx = range(len(spec.requests)) if requests is None else requests
    parts = []
    for i in idx:
        r = spec.requests[i]
        pos = torch.arange(r.c, r.c + r.n, dtype=torch.int64)
        parts.append(gen_block(spec.seed, KIND_Q, own_cid(spec, i), pos, spec.H_q, spec.d,
                               scale=spec.q_scale, device=device))
    if not parts:
        return torch.empty((0, spec.H_q, spec.d), dtype=torch.bfloat16, device=device)
    return torch.cat(parts, 0)


KIND_O, KIND_W = 3, 4


def matrix(seed: int, kind: int, tag: int, rows: int, cols: int, scale: float = 1.0, device="cpu") -> torch.Tensor:
    """A seeded bf16 [rows][cols] matrix (N(0,1)-scale, times ``scale``) from the
    same counter-based generator: the O_r / W_r inputs of the NEXT-4 projection."""
    pos = torch.arange(rows, dtype=torch.int64)
    return gen_block(seed, kind, tag, pos, 1, cols, scale=scale, device=device).reshape(rows, cols)
