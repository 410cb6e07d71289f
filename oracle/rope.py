"""Rotary position embedding (NEXT-4 prologue) for the oracle.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

The paper serves Llama-family models but never writes the
position encoding; the reading (R24) is the Llama rotate-half RoPE
with base theta over the first R dims, applied to Q and to K before K enters
the cache, the rotated values rounded to bf16 (the cache dtype):

    f_i = theta^(-2i/R),  a = p f_i,  i < R/2
    y[i]       = x[i] cos a - x[i + R/2] sin a
    y[i + R/2] = x[i + R/2] cos a + x[i] sin a
    y[i]       = x[i]                        (i >= R)

Pinned in tests/test_oracle_pins.py by what the rotation must satisfy:
position 0 is the identity, each (i, i + R/2) pair keeps its norm, the
2-D case is the rotation by p f_0 written with the textbook matrix, and
q(p + s) . k(p' + s) = q(p) . k(p') (the relative-position property).
"""
from __future__ import annotations

import numpy as np
import torch


def rope(x: np.ndarray, pos, theta: float, rot: int = 0) -> np.ndarray:
    """x float64 [n][H][d], pos int [n] -> rotated copy (fp64)."""
    x = np.asarray(x, dtype=np.float64)
    n, H, d = x.shape
    R = rot or d
    half = R // 2
    f = theta ** (-2.0 * np.arange(half, dtype=np.float64) / R)
    a = np.asarray(pos, dtype=np.float64)[:, None] * f[None, :]
    c = np.cos(a)[:, None, :]
    s = np.sin(a)[:, None, :]
    y = x.copy()
    x1, x2 = x[:, :, :half], x[:, :, half:R]
    y[:, :, :half] = x1 * c - x2 * s
    y[:, :, half:R] = x2 * c + x1 * s
    return y


def rope_bf16(x: torch.Tensor, pos, theta: float, rot: int = 0) -> torch.Tensor:
    """bf16 [n][H][d] -> bf16: the fp64 rotation rounded (RNE) to bf16."""
    y = rope(x.to(torch.float64).cpu().numpy(), pos, theta, rot)
    return torch.from_numpy(y).to(torch.bfloat16)
