"""Seeded physical placement of a BatchSpec in a paged pool, and the history
that must be in the cache before the iteration runs.

This is input *structure* (which physical block holds which logical block),
drawn as a seeded random permutation so tables are fragmented like a pool that
has seen churn (SURVEY.md §8(d) "physical block ids are fragmented").  It is
independent of the library allocator (hg_kv_alloc), which is checked
separately against oracle/mirror.py.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import List

import numpy as np


def _ceil_div(a: int, b: int) -> int:
    return -(-a // b)


@dataclass
class Layout:
    num_blocks: int
    block_table: np.ndarray      # int32 [R][W], -1 padded
    shared: np.ndarray           # int32 [R]: s_i
    group_blocks: dict           # group -> list of physical ids of its shared prefix


@dataclass
class AppendStep:
    """One history append: rows (table row, c, n, request index, content start)."""
    tables: List[List[int]]
    c: List[int]
    n: List[int]
    req: List[int]               # request whose content fills the rows


def make_layout(spec, seed: int = 0, slack: float = 0.05, num_blocks: int = None,
                width: int = None) -> Layout:
    rng = np.random.default_rng(7919 + seed)
    B = spec.B
    R = len(spec.requests)
    need_group = {}
    for i, r in enumerate(spec.requests):
        s = spec.shared_blocks(i)
        if s:
            need_group[r.group] = max(need_group.get(r.group, 0), s)
    priv = [_ceil_div(r.c + r.n, B) - spec.shared_blocks(i) for i, r in enumerate(spec.requests)]
    total = sum(need_group.values()) + sum(priv)
    if num_blocks is None:
        num_blocks = total + int(total * slack) + 16
    assert num_blocks >= total
    perm = rng.permutation(num_blocks).astype(np.int32)
    pos = 0
    gblocks = {}
    for g in sorted(need_group):
        gblocks[g] = [int(x) for x in perm[pos:pos + need_group[g]]]
        pos += need_group[g]
    W = max([_ceil_div(r.c + r.n, B) for r in spec.requests], default=1)
    W = max(W, width or 1)
    bt = np.full((R, W), -1, dtype=np.int32)
    shared = np.zeros(R, dtype=np.int32)
    for i, r in enumerate(spec.requests):
        s = spec.shared_blocks(i)
        row = (gblocks[r.group][:s] if s else []) + [int(x) for x in perm[pos:pos + priv[i]]]
        pos += priv[i]
        bt[i, :len(row)] = row
        shared[i] = s
    return Layout(num_blocks, bt, shared, gblocks)


def history_steps(spec, lay: Layout) -> List[AppendStep]:
    """Appends that fill the cache with every request's first c_i tokens.

    Step 0 writes each physically shared group prefix once (through a member's
    table); step 1 writes each request's private history [s_i*B, c_i).
    """
    B = spec.B
    steps = []
    first = {}
    for i, r in enumerate(spec.requests):
        s = spec.shared_blocks(i)
        if s and r.group not in first:
            first[r.group] = i
    if first:
        st = AppendStep([], [], [], [])
        for g, i in sorted(first.items()):
            s = spec.shared_blocks(i)
            st.tables.append([int(x) for x in lay.block_table[i]])
            st.c.append(0)
            st.n.append(s * B)
            st.req.append(i)
        steps.append(st)
    st = AppendStep([], [], [], [])
    for i, r in enumerate(spec.requests):
        lo = spec.shared_blocks(i) * B
        if r.c > lo:
            st.tables.append([int(x) for x in lay.block_table[i]])
            st.c.append(lo)
            st.n.append(r.c - lo)
            st.req.append(i)
    if st.c:
        steps.append(st)
    return steps
