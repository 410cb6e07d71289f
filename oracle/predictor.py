"""Batch-latency predictor of HyGen §4.2: features, OLS fit, predict, MAPE.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Eq. 1:  T = f(S_p, S_d, S_p^2, S_d^2, N_p, N_d)
Eq. 2:  T = f(S_p, S_d, S_p^2, N_p, N_d)
with f linear ("We employ linear regression").  S_p / S_d are the
total prefill / decode tokens, N_p / N_d the request counts.

Attention-exact extensions (readings R13-R15):
  P2    = sum over prefill requests of n_i (c_i + (n_i + 1) / 2)  (attended pairs)
  D_ctx = unique KV slots read by decode rows (a physically shared slot counted
          once, at any prefix depth: NEXT-3 / R23)

Feature order (index k, weight w[1 + k]; w[0] is the intercept):
  0 S_p, 1 S_d, 2 S_p2, 3 S_d2, 4 N_p, 5 N_d, 6 P2, 7 D_ctx
"""
from __future__ import annotations

import numpy as np

NAMES = ("S_p", "S_d", "S_p2", "S_d2", "N_p", "N_d", "P2", "D_ctx")
MASK_EQ1_IDENT = (1 << 0) | (1 << 2) | (1 << 3) | (1 << 4) | (1 << 5)  # Eq.1 minus collinear S_d
MASK_EQ2_IDENT = (1 << 0) | (1 << 2) | (1 << 4) | (1 << 5)            # Eq.2 minus collinear S_d
MASK_GRADED = (1 << 0) | (1 << 6) | (1 << 7) | (1 << 5) | (1 << 4)     # S_p, P2, D_ctx, N_d, N_p


def features(c, n, shared_tokens=None, group=None):
    """Feature vector of one batch.

    A row is decode iff n_i == 1 and c_i >= 1 (reading R5); every other row is
    prefill.  ``group[i]`` >= 0 with ``shared_tokens[i]`` marks physically
    shared prefixes for D_ctx."""
    R = len(c)
    S_p = S_d = N_p = N_d = 0
    P2 = 0.0
    D = 0
    seen = {}
    for i in range(R):
        ci, ni = int(c[i]), int(n[i])
        if ni == 1 and ci >= 1:
            N_d += 1
            S_d += 1
            D += ci + 1
            if group is not None and int(group[i]) >= 0:
                g = int(group[i])
                st = int(shared_tokens[i])
                if g in seen:
                    D -= st
                else:
                    seen[g] = st
        else:
            N_p += 1
            S_p += ni
            P2 += ni * (ci + (ni + 1) / 2.0)
    return np.array([S_p, S_d, float(S_p) ** 2, float(S_d) ** 2, N_p, N_d, P2, D], np.float64)


def features_paged(c, n, block_table, s, B: int):
    """The same features with D_ctx counted on the paged layout itself: the set
    of KV slots the decode rows read, a slot being (physical block, offset) for
    positions inside a row's s_i shared blocks and (row, position) otherwise."""
    f = features(c, n)
    slots = set()
    D = 0
    for i in range(len(c)):
        ci, ni = int(c[i]), int(n[i])
        if ni == 1 and ci >= 1:
            for p in range(ci + 1):
                if p < int(s[i]) * B:
                    slots.add((int(block_table[i][p // B]), p % B))
                else:
                    D += 1
    f[7] = D + len(slots)
    return f


def design(X, mask: int):
    cols = [k for k in range(8) if mask >> k & 1]
    X = np.asarray(X, np.float64).reshape(-1, 8)
    return np.hstack([np.ones((X.shape[0], 1)), X[:, cols]]), cols


def fit(X, y, mask: int, relative: bool = False):
    """OLS: minimise ||A w - y||_2 with A = [1, selected features].

    relative=True (HG_FIT_RELATIVE): minimise sum_i ((A w - y)_i / y_i)^2, i.e.
    the same regression with row i divided by y_i (weights 1 / y_i^2) -- the
    least-squares criterion nearest to the MAPE of P:414.  Needs y > 0."""
    A, cols = design(X, mask)
    y = np.asarray(y, np.float64)
    if relative:
        assert np.all(y > 0)
        A, y = A / y[:, None], np.ones_like(y)
    w_sel, *_ = np.linalg.lstsq(A, y, rcond=None)
    w = np.zeros(9)
    w[0] = w_sel[0]
    for k, col in enumerate(cols):
        w[1 + col] = w_sel[1 + k]
    return w


def predict(w, x):
    """w . [1, x] floored at 0."""
    return max(0.0, float(w[0] + np.dot(w[1:], np.asarray(x, np.float64))))


def mape(y_hat, y):
    y_hat, y = np.asarray(y_hat, np.float64), np.asarray(y, np.float64)
    return float(np.mean(np.abs(y_hat - y) / y))
