"""Integer mirror of the host-side steps: GET_NUM_BLOCKS, batch indices,
prefix groups, batch validation and the block allocator.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Written as straight-line
Python from the definitions; the library's outputs must match bit-exactly.
"""
from __future__ import annotations

from typing import Dict, List, Tuple

import numpy as np

# status codes of include/hygen.h (restated, not imported: the oracle shares no code)
OK, E_INVALID, E_OOM, E_SHARED_WRITE, E_RANK_DEFICIENT = 0, 1, 2, 3, 4


def get_num_blocks(tokens: int, block_size: int) -> int:
    """GET_NUM_BLOCKS(l) of Alg. 1: blocks needed for l tokens,
    ceil(l / B)."""
    if tokens <= 0:
        return 0
    q, r = divmod(tokens, block_size)
    return q + (1 if r else 0)


def batch_indices(block_table, c, n, s, B: int):
    """cu_q, kv_len, slot, prefix_group.

    cu_q[i+1] = cu_q[i] + n_i;  kv_len_i = c_i + n_i;
    slot[t] = bt[i][p // B] * B + p % B for p = c_i + j, t = cu_q[i] + j;
    prefix_group[i]: requests with s_i > 0 whose shared id sequences
    bt[i][0:s_i] are identical form a group, numbered by first appearance; -1
    when s_i == 0 (a.4, PSM "KV cache reuse through shared prefixes").
    """
    bt = np.asarray(block_table)
    R = len(c)
    cu = [0]
    for i in range(R):
        cu.append(cu[-1] + int(n[i]))
    kv_len = [int(c[i]) + int(n[i]) for i in range(R)]
    slot = []
    for i in range(R):
        for j in range(int(n[i])):
            p = int(c[i]) + j
            slot.append(int(bt[i][p // B]) * B + p % B)
    groups: Dict[Tuple[int, ...], int] = {}
    pg = []
    for i in range(R):
        if int(s[i]) > 0:
            key = tuple(int(x) for x in bt[i][:int(s[i])])
            if key not in groups:
                groups[key] = len(groups)
            pg.append(groups[key])
        else:
            pg.append(-1)
    return (np.array(cu, np.int32), np.array(kv_len, np.int32), np.array(slot, np.int64),
            np.array(pg, np.int32))


def validate(block_table, c, n, s, B: int, num_blocks: int, H_q: int = None, H_kv: int = None,
             append: bool = False) -> int:
    """Status the library must return for this batch (SURVEY §8(b) rules)."""
    bt = np.asarray(block_table)
    R = len(c)
    if H_q is not None and (H_kv is None or H_kv <= 0 or H_q <= 0 or H_q % H_kv):
        return E_INVALID
    owner: Dict[int, List[int]] = {}
    for i in range(R):
        if int(n[i]) < 1 or int(c[i]) < 0 or int(s[i]) < 0:
            return E_INVALID
        nb = get_num_blocks(int(c[i]) + int(n[i]), B)
        if nb > bt.shape[1] or int(s[i]) > nb:
            return E_INVALID
        row = [int(x) for x in bt[i][:nb]]
        if any(x < 0 or x >= num_blocks for x in row):
            return E_INVALID
        if len(set(row)) != len(row):
            return E_INVALID
        for col, x in enumerate(row):
            owner.setdefault(x, []).append((i, col))
    # an id used by several rows must sit inside every user's shared prefix
    for x, users in owner.items():
        if len(users) > 1:
            for (i, col) in users:
                if col >= int(s[i]):
                    return E_INVALID
    # shared prefixes form a trie (NEXT-3, R23): every row that shares
    # an id has it at the same column, after the same sequence of ids
    for x, users in owner.items():
        if len(users) > 1:
            i0, col0 = users[0]
            for (i, col) in users[1:]:
                if col != col0 or [int(y) for y in bt[i][:col]] != [int(y) for y in bt[i0][:col0]]:
                    return E_INVALID
    if append:
        for i in range(R):
            if int(c[i]) < int(s[i]) * B:
                return E_SHARED_WRITE
    return OK


class Allocator:
    """KV block allocator: all-or-nothing alloc of the smallest free ids in
    ascending order with refcount 1; retain += 1; release -= 1, freeing at 0
    (memory budget m of Alg. 1; conservation SPEC.md:175)."""

    def __init__(self, num_blocks: int):
        self.num_blocks = num_blocks
        self.ref = [0] * num_blocks

    def num_free(self) -> int:
        return sum(1 for r in self.ref if r == 0)

    def alloc(self, k: int):
        if k < 0:
            return E_INVALID, []
        free = [b for b in range(self.num_blocks) if self.ref[b] == 0]
        if k > len(free):
            return E_OOM, []
        out = free[:k]
        for b in out:
            self.ref[b] = 1
        return OK, out

    def retain(self, ids) -> int:
        if any(b < 0 or b >= self.num_blocks or self.ref[b] == 0 for b in ids):
            return E_INVALID
        for b in ids:
            self.ref[b] += 1
        return OK

    def release(self, ids) -> int:
        need: Dict[int, int] = {}
        for b in ids:
            if b < 0 or b >= self.num_blocks:
                return E_INVALID
            need[b] = need.get(b, 0) + 1
        if any(self.ref[b] < k for b, k in need.items()):
            return E_INVALID
        for b in ids:
            self.ref[b] -= 1
        return OK
