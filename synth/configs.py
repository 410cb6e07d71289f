"""Batch shapes for the BASELINE.json configs.

A request is (c, n): c tokens already cached, n new tokens this iteration
(decode iff n == 1), matching the paper's batch tuples (r, l, t_req) of
Alg. 1 and chunked prefill.  Shared-prefix
groups model PSM's "KV cache reuse through shared prefixes".

Nothing here computes attention or indexes the paged layout.
"""
from __future__ import annotations

from dataclasses import dataclass, field, replace
from typing import Dict, List, Optional, Tuple

import numpy as np

CONFIG_NAMES = ("toy_a", "toy_b", "c1", "c1_long", "c2", "c2_g8", "c2_none", "c2_private",
                "c2_nested", "c3", "p1", "p2")


@dataclass
class Request:
    c: int                    # cached tokens before this iteration (c_i)
    n: int                    # new tokens this iteration (n_i; 1 = decode)
    offline: bool = False     # HyGen tag: no numeric effect (reading R6)
    group: int = -1           # content group of the prefix (-1: none)
    prefix_tokens: int = 0    # tokens [0, prefix_tokens) carry the group's content
    share: bool = True        # prefix blocks physically shared (True) or private copies
    cid: int = -1             # own content id override (-1: request index)


@dataclass
class BatchSpec:
    name: str
    H_q: int
    H_kv: int
    d: int
    B: int
    seed: int
    requests: List[Request] = field(default_factory=list)
    q_scale: float = 1.0
    # nested prefix sharing (NEXT-3): child group -> (parent group, tokens of the
    # child's prefix that are the parent's); a member of the child holds the
    # parent's content on [0, split) and the child's on [split, prefix_tokens)
    group_parent: Dict[int, Tuple[int, int]] = field(default_factory=dict)
    # rotary embedding (NEXT-4 prologue): (theta, rotary_dim) or None; values from
    # synth are pre-rotary, the library / oracle rotate Q and K at their positions
    rope: Optional[Tuple[float, int]] = None

    @property
    def T(self) -> int:
        return sum(r.n for r in self.requests)

    @property
    def G_q(self) -> int:
        return self.H_q // self.H_kv

    def shared_blocks(self, i: int) -> int:
        """s_i: number of leading block-table entries that are physically shared."""
        r = self.requests[i]
        if r.group < 0 or not r.share:
            return 0
        return r.prefix_tokens // self.B

    def group_chain(self, g: int) -> List[Tuple[int, int]]:
        """[(group, start token)] from the root down to g: group k's content
        covers [start_k, start_{k+1})."""
        chain = [(g, 0)]
        while chain[0][0] in self.group_parent:
            parent, split = self.group_parent[chain[0][0]]
            chain[0] = (chain[0][0], split)
            chain.insert(0, (parent, 0))
        return chain

    def with_(self, **kw) -> "BatchSpec":
        return replace(self, **kw)


def shard_slice(spec: BatchSpec, G: int) -> BatchSpec:
    """One rank's slice of G-way KV-head sharding: H_kv / G KV heads
    and their H_q / G q heads, same requests (values of the first heads)."""
    assert spec.H_kv % G == 0
    return spec.with_(H_kv=spec.H_kv // G, H_q=spec.H_q // G)


def _uniform(rng, lo, hi, k):
    return [int(x) for x in rng.integers(lo, hi + 1, size=k)]


def make_config(name: str, seed: int = 0, q_scale: float = 1.0) -> BatchSpec:
    rng = np.random.default_rng(seed)
    if name in ("toy_a", "toy_b"):
        spec = BatchSpec(name, 2, 2, 64, 16, seed, q_scale=q_scale)
        if name == "toy_a":
            # r0 online prefill of 16 at c=0; r1, r2 offline decodes at c=32 sharing block S
            spec.requests = [Request(0, 16, False),
                             Request(32, 1, True, group=0, prefix_tokens=16),
                             Request(32, 1, True, group=0, prefix_tokens=16)]
        else:
            # r0 online chunk c=16,n=16 whose 16 cached tokens (block S) are shared with r1
            spec.requests = [Request(16, 16, False, group=0, prefix_tokens=16),
                             Request(32, 1, True, group=0, prefix_tokens=16),
                             Request(32, 1, True)]
        return spec
    if name in ("c1", "c1_long"):
        spec = BatchSpec(name, 32, 32, 128, 16, seed, q_scale=q_scale)
        c0 = 0 if name == "c1" else 3584
        reqs = [Request(c0, 512, False)]
        cs = _uniform(rng, 1024, 4096, 64)
        reqs += [Request(c, 1, k >= 32) for k, c in enumerate(cs)]
        spec.requests = reqs
        return spec
    if name.startswith("c2"):
        spec = BatchSpec(name, 32, 8, 128, 16, seed, q_scale=q_scale)
        cs = _uniform(rng, 2048, 8192, 256)
        reqs = []
        for k, c in enumerate(cs):
            if name == "c2":
                reqs.append(Request(c, 1, True, group=0, prefix_tokens=1024))
            elif name == "c2_g8":
                reqs.append(Request(c, 1, True, group=k // 32, prefix_tokens=1024))
            elif name == "c2_nested":
                # NEXT-3: one 1024-token system prefix shared by all 256 (group 8),
                # then 8 few-shot blocks of 512 tokens shared by 32 each (groups 0-7)
                reqs.append(Request(c, 1, True, group=k // 32, prefix_tokens=1536))
            elif name == "c2_private":
                reqs.append(Request(c, 1, True, group=0, prefix_tokens=1024, share=False))
            else:
                reqs.append(Request(c, 1, True))
        spec.requests = reqs
        if name == "c2_nested":
            spec.group_parent = {g: (8, 1024) for g in range(8)}
        return spec
    if name == "c3":
        spec = BatchSpec(name, 64, 8, 128, 16, seed, q_scale=q_scale)
        reqs = [Request(0, 512, False)]
        reqs += [Request(c, 1, False) for c in _uniform(rng, 1024, 8192, 128)]
        reqs += [Request(c, 1, True, group=k // 32, prefix_tokens=1024)
                 for k, c in enumerate(_uniform(rng, 1024, 8192, 128))]
        spec.requests = reqs
        return spec
    if name == "p1":
        spec = BatchSpec(name, 32, 32, 128, 16, seed, q_scale=q_scale)
        spec.requests = [Request(c, 512, k >= 2) for k, c in enumerate((0, 2048, 4096, 6144))]
        return spec
    if name == "p2":
        spec = BatchSpec(name, 32, 32, 128, 16, seed, q_scale=q_scale)
        spec.requests = [Request(6144, 2048, True)]
        return spec
    raise ValueError(f"unknown config {name}")


def make_fuzz(seed: int, d: int = None, G_q: int = None, H_kv: int = None, B: int = 16) -> BatchSpec:
    """Random small batch (SURVEY.md §8(c.6) fuzz row): R<=16, c<=300, n<=40, random groups."""
    rng = np.random.default_rng(10_000 + seed)
    d = d if d is not None else int(rng.choice([64, 128]))
    G_q = G_q if G_q is not None else int(rng.choice([1, 4, 8]))
    H_kv = H_kv if H_kv is not None else int(rng.choice([1, 2]))
    spec = BatchSpec(f"fuzz{seed}", G_q * H_kv, H_kv, d, B, seed)
    R = int(rng.integers(1, 17))
    ngroups = int(rng.integers(0, 3))
    gprefix = [int(rng.integers(1, 6)) * B for _ in range(ngroups)]
    reqs = []
    for k in range(R):
        g = int(rng.integers(-1, ngroups)) if ngroups else -1
        if g >= 0:
            pt = gprefix[g]
            c = pt + int(rng.integers(0, 200))
        else:
            pt = 0
            c = int(rng.integers(0, 301))
        n = 1 if (rng.random() < 0.5 and c > 0) else int(rng.integers(1, 41))
        reqs.append(Request(c, n, bool(rng.random() < 0.5), group=g, prefix_tokens=pt))
    spec.requests = reqs
    return spec


def make_fuzz_nested(seed: int, d: int = None, G_q: int = None, H_kv: int = None, B: int = 16) -> BatchSpec:
    """Random small batch with a prefix trie of depth <= 3 (NEXT-3): roots, children
    and grandchildren groups with block-aligned splits; members at every level,
    prefill rows among them, and rows without sharing."""
    rng = np.random.default_rng(20_000 + seed)
    d = d if d is not None else int(rng.choice([64, 128]))
    G_q = G_q if G_q is not None else int(rng.choice([1, 4, 8]))
    H_kv = H_kv if H_kv is not None else int(rng.choice([1, 2]))
    spec = BatchSpec(f"nfuzz{seed}", G_q * H_kv, H_kv, d, B, seed)
    # groups: (tokens of the whole prefix), parents with their split
    plen, parent = {}, {}
    ng = 0
    for _ in range(int(rng.integers(1, 3))):           # roots
        root = ng
        plen[root] = int(rng.integers(1, 5)) * B
        ng += 1
        for _ in range(int(rng.integers(0, 3))):       # children
            ch = ng
            plen[ch] = plen[root] + int(rng.integers(1, 4)) * B
            parent[ch] = (root, plen[root])
            ng += 1
            for _ in range(int(rng.integers(0, 2))):   # grandchildren
                gc = ng
                plen[gc] = plen[ch] + int(rng.integers(1, 3)) * B
                parent[gc] = (ch, plen[ch])
                ng += 1
    reqs = []
    for k in range(int(rng.integers(2, 20))):
        g = int(rng.integers(-1, ng))
        if g >= 0:
            pt = plen[g]
            c = pt + int(rng.integers(0, 150))
        else:
            pt = 0
            c = int(rng.integers(0, 301))
        n = 1 if (rng.random() < 0.7 and c > 0) else int(rng.integers(1, 41))
        reqs.append(Request(c, n, bool(rng.random() < 0.5), group=g, prefix_tokens=pt))
    spec.requests = reqs
    spec.group_parent = parent
    return spec
