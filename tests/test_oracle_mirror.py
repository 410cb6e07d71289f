"""Pins for oracle/mirror.py and oracle/predictor.py (CPU)."""
import json
import os
import time

import numpy as np
import pytest

from oracle import mirror
from oracle import predictor as P

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def test_get_num_blocks_spec_examples():
    for l, B, exp in gold("spec_examples.json")["get_num_blocks"]["cases"]:
        assert mirror.get_num_blocks(l, B) == exp


def test_get_num_blocks_brute():
    for B in (1, 3, 16):
        for l in range(0, 100):
            assert mirror.get_num_blocks(l, B) == len(range(0, l, B))


def test_allocator_script():
    g = gold("allocator_script.json")
    a = mirror.Allocator(g["num_blocks"])
    for st in g["steps"]:
        if st["op"] == "alloc":
            s, ids = a.alloc(st["n"])
            assert (s, ids) == (st["status"], st["ids"])
        elif st["op"] == "retain":
            assert a.retain(st["ids"]) == st["status"]
        else:
            assert a.release(st["ids"]) == st["status"]
        assert a.num_free() == st["free"]


def test_allocator_conservation_random():
    rng = np.random.default_rng(0)
    a = mirror.Allocator(64)
    held = []   # one entry per outstanding reference
    for _ in range(2000):
        op = rng.integers(0, 3)
        if op == 0:
            s, ids = a.alloc(int(rng.integers(0, 9)))
            if s == 0:
                held += ids
        elif op == 1 and held:
            b = held[int(rng.integers(0, len(held)))]
            assert a.retain([b]) == 0
            held.append(b)
        elif held:
            b = held.pop(int(rng.integers(0, len(held))))
            assert a.release([b]) == 0
        assert a.num_free() + len(set(held)) == 64


def test_batch_indices_hand_example():
    # two requests, B=4: r0 c=5 n=3 table [7,2,9]; r1 c=0 n=2 table [4]; r2 decode sharing [7]
    bt = [[7, 2, 9], [4, -1, -1], [7, 3, -1]]
    cu, kv, slot, pg = mirror.batch_indices(bt, [5, 0, 4], [3, 2, 1], [1, 0, 1], 4)
    assert cu.tolist() == [0, 3, 5, 6]
    assert kv.tolist() == [8, 2, 5]
    # p=5,6,7 -> block 2 offs 1,2,3 ; p=0,1 -> block 4 ; p=4 -> block 3 off 0
    assert slot.tolist() == [2 * 4 + 1, 2 * 4 + 2, 2 * 4 + 3, 16, 17, 12]
    assert pg.tolist() == [0, -1, 0]


def test_validate_rules():
    B, N = 4, 16
    ok = dict(block_table=[[0, 1], [0, 2]], c=[4, 5], n=[1, 1], s=[1, 1])
    assert mirror.validate(B=B, num_blocks=N, **ok) == 0
    assert mirror.validate([[0, 1], [0, 2]], [4, 5], [0, 1], [1, 1], B, N) == mirror.E_INVALID
    assert mirror.validate([[0, 1], [0, 2]], [4, 5], [1, 1], [0, 1], B, N) == mirror.E_INVALID
    assert mirror.validate([[0, 16]], [4], [1], [0], B, N) == mirror.E_INVALID
    assert mirror.validate([[3, 3]], [4], [1], [0], B, N) == mirror.E_INVALID
    assert mirror.validate([[0, 1], [0, 2]], [3, 5], [1, 1], [1, 1], B, N, append=True) == mirror.E_SHARED_WRITE
    # nested sharing (NEXT-3, R23): a common root block, then different children: valid
    assert mirror.validate([[0, 1, 5], [0, 2, 6]], [9, 9], [1, 1], [2, 2], B, N) == 0
    assert mirror.validate([[0, 1, 5], [0, 1, 6], [0, 7, 8]], [9, 9, 9], [1, 1, 1], [2, 2, 1], B, N) == 0
    # not a trie: a shared id at different columns, or after different ids
    assert mirror.validate([[0, 1, 5], [1, 0, 6]], [9, 9], [1, 1], [2, 2], B, N) == mirror.E_INVALID
    assert mirror.validate([[0, 1, 5], [2, 1, 6]], [9, 9], [1, 1], [2, 2], B, N) == mirror.E_INVALID
    # a block inside one row's shared prefix but private in another
    assert mirror.validate([[0, 1, 5], [0, 2, 1]], [9, 9], [1, 1], [2, 1], B, N) == mirror.E_INVALID
    assert mirror.validate([[0, 1]], [4], [1], [0], B, N, H_q=6, H_kv=4) == mirror.E_INVALID


def test_featurize_spec_examples():
    for case in gold("spec_examples.json")["featurize"]["cases"]:
        f = P.features(case["c"], case["n"])
        assert f[:6].tolist() == case["expect"]


def test_predict_spec_example():
    g = gold("spec_examples.json")["predict_affine"]
    w = np.zeros(9)
    w[0] = g["intercept"]
    for k, name in enumerate(P.NAMES):
        w[1 + k] = g["weights"].get(name, 0.0)
    x = np.array([g["features"].get(nm, 0) for nm in P.NAMES], float)
    assert abs(P.predict(w, x) - g["expected_ms"]) < 1e-12
    assert P.predict(np.r_[-5.0, np.zeros(8)], x * 0) == 0.0


def test_p2_and_dctx_closed_forms():
    # single chunk at c=0: P2 = n(n+1)/2 = S_p^2/2 + S_p/2
    f = P.features([0], [100])
    assert f[6] == 100 * 101 / 2 == f[2] / 2 + f[0] / 2
    # decode rows of one group sharing 64 tokens: D_ctx = sum(c+1) - (k-1)*64
    f = P.features([100, 200, 300], [1, 1, 1], shared_tokens=[64] * 3, group=[0, 0, 0])
    assert f[7] == 101 + 201 + 301 - 2 * 64


def _synthetic(n, rng, w_true, mask, noise=0.0):
    X = []
    for _ in range(n):
        R = int(rng.integers(1, 40))
        c = rng.integers(0, 4000, R)
        nn = np.where(rng.random(R) < 0.7, 1, rng.integers(2, 600, R))
        c = np.where((nn == 1) & (c == 0), 1, c)
        X.append(P.features(c, nn))
    X = np.array(X)
    A, cols = P.design(X, mask)
    y = A @ np.r_[w_true[0], w_true[1:][cols]]
    return X, y * (1 + noise * rng.standard_normal(n))


def test_fit_recovers_noise_free():
    rng = np.random.default_rng(1)
    w_true = np.array([0.02, 1e-4, 0, 2e-9, 0, 3e-3, 1e-3, 5e-8, 4e-6])
    X, y = _synthetic(500, rng, w_true, P.MASK_GRADED)
    w = P.fit(X, y, P.MASK_GRADED)
    _, cols = P.design(X, P.MASK_GRADED)
    np.testing.assert_allclose(w[[0] + [1 + c for c in cols]], w_true[[0] + [1 + c for c in cols]],
                               rtol=1e-7)
    assert P.mape([P.predict(w, x) for x in X], y) < 1e-9


def test_fit_noisy_heldout_mape():
    rng = np.random.default_rng(2)
    w_true = np.array([0.5, 1e-3, 0, 2e-7, 0, 3e-2, 1e-2, 0, 0])
    X, y = _synthetic(2000, rng, w_true, P.MASK_EQ2_IDENT, noise=0.01)
    w = P.fit(X[:1600], y[:1600], P.MASK_EQ2_IDENT)
    assert P.mape([P.predict(w, x) for x in X[1600:]], y[1600:]) < 0.02


# ---- relative-error fit (HG_FIT_RELATIVE) ------------------------------------------
def test_relative_fit_intercept_only_closed_form():
    """mask 0: minimise sum (w0 / y_i - 1)^2  =>  w0 = sum(1/y) / sum(1/y^2)."""
    rng = np.random.default_rng(3)
    y = rng.uniform(0.05, 3.0, 200)
    X = np.zeros((200, 8))
    w = P.fit(X, y, 0, relative=True)
    assert abs(w[0] - np.sum(1 / y) / np.sum(1 / y ** 2)) < 1e-12 * w[0]
    assert abs(P.fit(X, y, 0)[0] - y.mean()) < 1e-12   # OLS: the mean


def test_relative_fit_noise_free_and_scale_invariant():
    rng = np.random.default_rng(11)
    X = np.abs(rng.standard_normal((300, 8))) * [100, 1, 1e4, 1, 3, 5, 1e5, 1e4]
    A, cols = P.design(X, P.MASK_GRADED)
    wt = np.r_[0.03, np.abs(rng.standard_normal(len(cols))) * 1e-5]
    y = A @ wt
    w = P.fit(X, y, P.MASK_GRADED, relative=True)
    np.testing.assert_allclose(np.r_[w[0], w[1:][cols]], wt, rtol=1e-8)
    yn = y * (1 + 0.05 * rng.standard_normal(300))
    w1 = P.fit(X, yn, P.MASK_GRADED, relative=True)
    w2 = P.fit(X, 7.0 * yn, P.MASK_GRADED, relative=True)
    np.testing.assert_allclose(w2, 7.0 * w1, rtol=1e-9, atol=1e-18)


def test_relative_fit_optimal_for_its_criterion():
    """Each fit is optimal under its own criterion: the relative fit has the
    smaller sum of squared relative errors, OLS the smaller sum of squares."""
    rng = np.random.default_rng(12)
    X = np.abs(rng.standard_normal((400, 8))) * 50
    y = 0.02 + X @ np.abs(rng.standard_normal(8)) * 1e-3
    y = y * np.exp(0.2 * rng.standard_normal(400))
    wr = P.fit(X, y, P.MASK_GRADED, relative=True)
    wo = P.fit(X, y, P.MASK_GRADED)
    pr = np.array([wr[0] + wr[1:] @ x for x in X])
    po = np.array([wo[0] + wo[1:] @ x for x in X])
    assert np.sum(((pr - y) / y) ** 2) <= np.sum(((po - y) / y) ** 2)
    assert np.sum((po - y) ** 2) <= np.sum((pr - y) ** 2)
    # small perturbations of the relative solution never lower its criterion
    for k in range(20):
        d = wr + rng.standard_normal(9) * 1e-3 * (np.abs(wr) + 1e-12) * (np.r_[1, [(P.MASK_GRADED >> i) & 1 for i in range(8)]])
        pd = np.array([d[0] + d[1:] @ x for x in X])
        assert np.sum(((pd - y) / y) ** 2) >= np.sum(((pr - y) / y) ** 2) - 1e-12
