"""Dense brute-force attention on *logical* (unpaged) sequences, numpy fp64.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Used to pin oracle.c on
tiny inputs: it never looks at a block table, so a paging / slot / offset bug
in oracle.c cannot be mirrored here.

softmax(Q K^T / sqrt(d) + M) V with M[j, p] = 0 if p <= c + j else -inf
(causal alignment to absolute positions, reading R3; scale 1/sqrt(d),
reading R1; GQA head map h -> h // (H_q/H_kv), reading R4).
"""
from __future__ import annotations

import numpy as np


def attention_dense(q, K, V, c: int):
    """q [n][H_q][d], K/V [L][H_kv][d] (L >= c + n), any float dtype -> fp64.

    Returns (O [n][H_q][d], LSE [n][H_q])."""
    q = np.asarray(q, np.float64)
    K = np.asarray(K, np.float64)
    V = np.asarray(V, np.float64)
    n, H_q, d = q.shape
    H_kv = K.shape[1]
    G = H_q // H_kv
    L = c + n
    out = np.zeros((n, H_q, d))
    lse = np.zeros((n, H_q))
    j = np.arange(n)[:, None]
    p = np.arange(L)[None, :]
    mask = np.where(p <= c + j, 0.0, -np.inf)
    for h in range(H_q):
        g = h // G
        S = q[:, h, :] @ K[:L, g, :].T / np.sqrt(d) + mask
        m = S.max(axis=1, keepdims=True)
        P = np.exp(S - m)
        l = P.sum(axis=1, keepdims=True)
        out[:, h, :] = (P @ V[:L, g, :]) / l
        lse[:, h] = (m + np.log(l))[:, 0]
    return out, lse
