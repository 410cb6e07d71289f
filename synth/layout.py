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
    shared: List[int]            # s of each row (its blocks before c that are shared)
    group: List[int]             # group prefix a row writes (-1: private history)


def _group_needs(spec):
    """Blocks each group's physical prefix must span, and a request whose content
    fills them: a member's own s_i, or the split where a child group starts
    (nested sharing, NEXT-3).  Returns ({group: blocks}, {group: request}, {group: depth})."""
    B = spec.B
    need, src, depth = {}, {}, {}
    for i, r in enumerate(spec.requests):
        s = spec.shared_blocks(i)
        if not s:
            continue
        chain = spec.group_chain(r.group)
        for k, (g, _) in enumerate(chain):
            nb = chain[k + 1][1] // B if k + 1 < len(chain) else s
            depth[g] = k
            if nb > need.get(g, 0):
                need[g], src[g] = nb, i
    return need, src, depth


def make_layout(spec, seed: int = 0, slack: float = 0.05, num_blocks: int = None,
                width: int = None) -> Layout:
    rng = np.random.default_rng(7919 + seed)
    B = spec.B
    R = len(spec.requests)
    need, _, depth = _group_needs(spec)
    own = {}   # blocks a group adds beyond its parent's split
    for g, nb in need.items():
        split = spec.group_parent[g][1] // B if g in spec.group_parent else 0
        own[g] = nb - split
    priv = [_ceil_div(r.c + r.n, B) - spec.shared_blocks(i) for i, r in enumerate(spec.requests)]
    total = sum(own.values()) + sum(priv)
    if num_blocks is None:
        num_blocks = total + int(total * slack) + 16
    assert num_blocks >= total
    perm = rng.permutation(num_blocks).astype(np.int32)
    pos = 0
    gblocks = {}
    for g in sorted(need, key=lambda x: (depth[x], x)):   # parents before children
        base = []
        if g in spec.group_parent:
            parent, split = spec.group_parent[g]
            base = gblocks[parent][:split // B]
        gblocks[g] = base + [int(x) for x in perm[pos:pos + own[g]]]
        pos += own[g]
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

    First each physically shared group prefix is written once, one step per
    trie depth (a child's rows list its parent's blocks as their shared prefix
    and write only the child's own blocks), through pseudo rows whose table is
    the group's block list; then each request's private history [s_i*B, c_i).
    """
    B = spec.B
    steps = []
    need, src, depth = _group_needs(spec)
    W = lay.block_table.shape[1]
    for dep in sorted(set(depth.values())):
        st = AppendStep([], [], [], [], [], [])
        for g in sorted(x for x in need if depth[x] == dep):
            split = spec.group_parent[g][1] if g in spec.group_parent else 0
            if need[g] * B <= split:
                continue
            row = lay.group_blocks[g][:need[g]]
            st.tables.append(row + [-1] * (W - len(row)))
            st.c.append(split)
            st.n.append(need[g] * B - split)
            st.req.append(src[g])
            st.shared.append(split // B)
            st.group.append(g)
        if st.c:
            steps.append(st)
    st = AppendStep([], [], [], [], [], [])
    for i, r in enumerate(spec.requests):
        lo = spec.shared_blocks(i) * B
        if r.c > lo:
            st.tables.append([int(x) for x in lay.block_table[i]])
            st.c.append(lo)
            st.n.append(r.c - lo)
            st.req.append(i)
            st.shared.append(spec.shared_blocks(i))
            st.group.append(-1)
    if st.c:
        steps.append(st)
    return steps
