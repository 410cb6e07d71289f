"""Plain mirror of PSM and Alg. 3.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  The prefix tree is nested
dicts (insertion-ordered); DFS is recursive; the shared-prefix length of each
request with its DFS predecessor is computed by comparing the two token lists
directly (not through the tree).
"""
from __future__ import annotations

from . import scheduler as S


class Trie:
    def __init__(self):
        self.root = {"kids": {}, "reqs": []}
        self.tokens = {}

    def insert(self, rid, tokens):
        node = self.root
        for tok in tokens:
            node = node["kids"].setdefault(tok, {"kids": {}, "reqs": []})
        node["reqs"].append(rid)
        self.tokens[rid] = list(tokens)

    def remove(self, rid):
        path = [self.root]
        toks = self.tokens.pop(rid)
        for tok in toks:
            path.append(path[-1]["kids"][tok])
        path[-1]["reqs"].remove(rid)
        # prune the subtree the removal emptied (reading R22: children keep their
        # order of first insertion into the live tree)
        for depth in range(len(toks), 0, -1):
            node = path[depth]
            if node["reqs"] or node["kids"]:
                break
            del path[depth - 1]["kids"][toks[depth - 1]]

    def dfs(self):
        out = []

        def walk(node):
            out.extend(node["reqs"])
            for child in node["kids"].values():
                walk(child)
        walk(self.root)
        return out

    def lcp_with_prev(self):
        order = self.dfs()
        res = []
        for k, rid in enumerate(order):
            if k == 0:
                res.append(0)
                continue
            a, b = self.tokens[order[k - 1]], self.tokens[rid]
            n = 0
            while n < min(len(a), len(b)) and a[n] == b[n]:
                n += 1
            res.append(n)
        return order, res


def offline_schedule(w, block_size, trie, running, by_id, t, c, m, batch=None):
    """Alg. 3 with the readings of oracle/scheduler.py; decode gate `t < t_req => break` (R16).
    batch: the iteration's batch so far (the online phase's entries), as in
    scheduler.schedule; extended in place."""
    if batch is None:
        batch = []
    if ("w0",) not in batch:
        t = t - w[0]
        batch.append(("w0",))
    B, out = batch, []

    def marg(e):
        return max(0.0, S._lin(w, S._features(B + [e])) - S._lin(w, S._features(B)))

    def max_prefill(r):
        ci, left, st, g = r
        for cand in range(min(c, left, m * block_size), 0, -1):
            tr = marg(("p", ci, cand, g, st))
            if tr <= t:
                return cand, tr
        return 0, 0.0

    for i, r in enumerate(running):
        ci, left, st, g = r
        if left <= 0:
            e = ("d", ci, 1, g, st)
            tr = marg(e)
            if t < tr:
                return out, t, c, m
            t -= tr
            B.append(e)
            out.append((i, 0, tr))
        else:
            l, tr = max_prefill(r)
            if l <= 0:
                return out, t, c, m
            B.append(("p", ci, l, g, st))
            t -= tr
            c -= l
            m -= S._num_blocks(l, block_size)
            out.append((i, l, tr))
    while trie.dfs():
        rid = trie.dfs()[0]
        l, tr = max_prefill(by_id[rid])
        if l <= 0:
            break
        ci, left, st, g = by_id[rid]
        B.append(("p", ci, l, g, st))
        t -= tr
        c -= l
        m -= S._num_blocks(l, block_size)
        out.append((len(running) + rid, l, tr))
        trie.remove(rid)
    return out, t, c, m
