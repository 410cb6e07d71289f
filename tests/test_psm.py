"""PSM prefix tree and Alg. 3 (NEXT-2) against the paper's worked example
 and the plain mirror oracle/psm.py (CPU)."""
import json
import os

import numpy as np
import pytest

import paper_2501_14808_b200 as hg
from oracle import psm as OP

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "psm_example.json")))


def test_paper_worked_example():
    t = hg.PrefixTree()
    for rid, toks in enumerate(GOLD["queue"]):
        t.hg_psm_insert(rid, toks)
    order, lcp = t.hg_psm_dfs_order()
    assert order == GOLD["psm_order"] and lcp == GOLD["lcp_with_prev"]
    batches = [order[k:k + 2] for k in range(0, len(order), 2)]
    assert batches == GOLD["psm_batches_of_two"]
    fcfs = [list(range(len(GOLD["queue"])))[k:k + 2] for k in range(0, 4, 2)]
    assert fcfs == GOLD["fcfs_batches_of_two"]
    # FCFS pairs share nothing; PSM pairs share two tokens each
    share = lambda a, b: len(os.path.commonprefix([GOLD["queue"][a], GOLD["queue"][b]]))
    assert [share(*b) for b in fcfs] == [0, 0] and [share(*b) for b in batches] == [2, 2]


@pytest.mark.parametrize("seed", range(60))
def test_dfs_order_and_lcp_match_mirror(seed):
    rng = np.random.default_rng(seed)
    t, m = hg.PrefixTree(), OP.Trie()
    n = int(rng.integers(1, 60))
    stems = [list(rng.integers(0, 5, int(rng.integers(0, 6)))) for _ in range(6)]
    ids = list(range(n))
    for rid in ids:
        toks = stems[int(rng.integers(0, 6))] + list(rng.integers(0, 4, int(rng.integers(0, 5))))
        t.hg_psm_insert(rid, toks)
        m.insert(rid, toks)
    for rid in rng.permutation(n)[: n // 3]:
        t.hg_psm_remove(int(rid))
        m.remove(int(rid))
    got = t.hg_psm_dfs_order()
    exp = m.lcp_with_prev()
    assert got[0] == exp[0] and got[1] == exp[1]
    assert t.hg_psm_size() == len(exp[0])


def test_errors():
    t = hg.PrefixTree()
    t.hg_psm_insert(0, [1, 2])
    assert hg.status_of(t.hg_psm_insert, 0, [3]) == hg.HG_E_INVALID
    assert hg.status_of(t.hg_psm_remove, 5) == hg.HG_E_INVALID
    t.hg_psm_insert(1, [])                      # empty prompt sits at the root: first in DFS
    assert t.hg_psm_dfs_order()[0] == [1, 0]


def _model(w):
    mm = hg.hg_predictor()
    for k, v in enumerate(w):
        mm.w[k] = v
    return mm


@pytest.mark.parametrize("seed", range(120))
def test_offline_schedule_matches_mirror(seed):
    rng = np.random.default_rng(500 + seed)
    w = list(np.abs(rng.standard_normal(9)) * np.array([0.05, 1e-3, 1e-3, 1e-7, 1e-4, 0.02, 0.01, 1e-7, 5e-6]))
    running = []
    for _ in range(int(rng.integers(0, 8))):
        left = 0 if rng.random() < 0.6 else int(rng.integers(1, 2000))
        running.append((int(rng.integers(1, 5000)), left, 0, -1))
    n_ids = int(rng.integers(0, 20))
    by_id = [(0, int(rng.integers(1, 3000)), 0, -1) for _ in range(n_ids)]
    tree, mt = hg.PrefixTree(), OP.Trie()
    for rid in range(n_ids):
        toks = list(rng.integers(0, 3, int(rng.integers(0, 5))))
        tree.hg_psm_insert(rid, toks)
        mt.insert(rid, toks)
    t, c, m = float(rng.uniform(0.05, 2.0)), int(rng.integers(0, 4096)), int(rng.integers(0, 500))
    got = hg.hg_psm_offline_schedule(_model(w), tree, running, by_id, t, c, m)
    exp = OP.offline_schedule(w, 16, mt, running, by_id, t, c, m)
    assert [(a, b) for a, b, _ in got[0]] == [(a, b) for a, b, _ in exp[0]]
    np.testing.assert_allclose([x for _, _, x in got[0]], [x for _, _, x in exp[0]], rtol=1e-9, atol=1e-12)
    assert got[2:] == exp[2:] and abs(got[1] - exp[1]) < 1e-9
    assert tree.hg_psm_size() == len(mt.dfs())


@pytest.mark.parametrize("seed", range(40))
def test_interleaved_ops_match_mirror(seed):
    """Inserts, removals (which prune emptied subtrees) and DFS reads interleaved:
    a request inserted into a pruned subtree's place goes after its live siblings
    in both the library and the mirror (R22), and the LCP of live neighbours
    separated by removed entries is recomputed correctly."""
    rng = np.random.default_rng(900 + seed)
    t, m = hg.PrefixTree(), OP.Trie()
    alive, nxt = [], 0
    stems = [list(rng.integers(0, 4, int(rng.integers(0, 5)))) for _ in range(5)]
    for step in range(120):
        op = rng.random()
        if op < 0.5 or not alive:
            toks = stems[int(rng.integers(0, 5))] + list(rng.integers(0, 3, int(rng.integers(0, 4))))
            t.hg_psm_insert(nxt, toks)
            m.insert(nxt, toks)
            alive.append(nxt)
            nxt += 1
        elif op < 0.85:
            rid = alive.pop(int(rng.integers(0, len(alive))))
            t.hg_psm_remove(rid)
            m.remove(rid)
        else:   # Alg. 3's loop: take the next DFS request and remove it
            ids, _ = t.hg_psm_dfs_order(1)
            assert ids == m.dfs()[:1]
            t.hg_psm_remove(ids[0])
            m.remove(ids[0])
            alive.remove(ids[0])
        k = int(rng.integers(1, 8))
        got = t.hg_psm_dfs_order(k)
        order, lcp = m.lcp_with_prev()
        assert got == (order[:k], lcp[:k]), step
        assert t.hg_psm_size() == len(alive)


def test_admission_loop_is_linear():
    """P:647-651 (O(1) next request): admitting 2,048 offline requests with 1,024-token
    shared prefixes one at a time (dfs_order(1) then remove, as Alg. 3 does) must not
    rebuild the tree per removal -- bounded wall time (the quadratic version took
    minutes at this size)."""
    import time
    rng = np.random.default_rng(3)
    t = hg.PrefixTree()
    for g in range(64):
        prefix = list(rng.integers(0, 32000, 1024))
        for k in range(32):
            t.hg_psm_insert(g * 32 + k, prefix + list(rng.integers(0, 32000, 64)))
    t0 = time.perf_counter()
    seen = []
    while t.hg_psm_size():
        ids, _ = t.hg_psm_dfs_order(1)
        seen.append(ids[0])
        t.hg_psm_remove(ids[0])
    assert sorted(seen) == list(range(2048))
    assert time.perf_counter() - t0 < 2.0
