"""Output projection + reduce-scatter of a tensor-parallel attention layer
 for the oracle.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Rank r holds O_r [T][K_r] and the rows W_r [K_r][N] of the projection that
match its heads; the layer output is Y = sum_r O_r W_r, and the reduce-scatter
gives rank o the token rows [o T // G, (o + 1) T // G).  fp64 throughout; the
matrix product is numpy's (a library primitive used as a step).  Pinned in
tests/test_oracle_pins.py by a triple loop on tiny sizes and by the block
identity sum_r O_r W_r = [O_0 .. O_{G-1}] [W_0; ..; W_{G-1}].
"""
from __future__ import annotations

import numpy as np


def shard_rows(T: int, G: int, o: int):
    return (o * T) // G, ((o + 1) * T) // G


def out_proj_rs(O_list, W_list):
    """O_list[r] [T][K_r], W_list[r] [K_r][N] (any float) -> [Y shard of rank o] (fp64)."""
    G = len(O_list)
    T = np.asarray(O_list[0]).shape[0]
    Y = sum(np.asarray(O, np.float64) @ np.asarray(W, np.float64) for O, W in zip(O_list, W_list))
    return [Y[slice(*shard_rows(T, G, o))] for o in range(G)]
