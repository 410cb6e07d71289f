"""Run the oracle end to end on a synth BatchSpec.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Inputs come only from the
seeded generators in ``synth`` (never from the CUDA path):
  1. history appends fill each request's first c_i tokens (shared group
     prefixes written once), 2. the iteration's append writes the n_i new
     tokens, 3. attention for the selected requests.
"""
from __future__ import annotations

import numpy as np
import torch

from synth.layout import history_steps, make_layout
from synth.values import KIND_K, KIND_V, kv_values, q_values

from . import OraclePool
from .rope import rope_bf16


def _k(spec, i, c0, c1, device):
    """K rows of request i at positions [c0, c1) as the cache holds them (rotated when spec.rope)."""
    k = kv_values(spec, i, c0, c1, KIND_K, device).cpu()
    if getattr(spec, "rope", None):
        k = rope_bf16(k, np.arange(c0, c1), *spec.rope)
    return k


def fill_pool(spec, lay, req_sel=None, pool=None, device="cpu"):
    """Oracle pool holding history + the iteration's new tokens.

    With ``req_sel`` only those requests (and their shared group prefixes) are
    written: a full-size pool stays lazily mapped except for the sampled blocks.
    ``device`` only selects where synth evaluates its counter-based generator
    (bit-identical on CPU and CUDA, tests/test_gpu_parity.py); values are
    copied to host memory before the oracle sees them.
    """
    pool = pool or OraclePool(lay.num_blocks, spec.H_kv, spec.B, spec.d)
    sel = None if req_sel is None else set(int(i) for i in req_sel)
    for st in history_steps(spec, lay):
        rows = [k for k, i in enumerate(st.req)
                if sel is None or (st.group[k] < 0 and i in sel) or
                (st.group[k] >= 0 and _group_needed(spec, st.group[k], sel))]
        if not rows:
            continue
        ks, vs = [], []
        for k in rows:
            i = st.req[k]
            ks.append(_k(spec, i, st.c[k], st.c[k] + st.n[k], device))
            vs.append(kv_values(spec, i, st.c[k], st.c[k] + st.n[k], KIND_V, device).cpu())
        pool.append([st.tables[k] for k in rows], [st.c[k] for k in rows],
                     [st.n[k] for k in rows], torch.cat(ks), torch.cat(vs))
    idx = [i for i in range(len(spec.requests)) if sel is None or i in sel]
    if idx:
        ks = torch.cat([_k(spec, i, spec.requests[i].c, spec.requests[i].c + spec.requests[i].n, device)
                        for i in idx])
        vs = torch.cat([kv_values(spec, i, spec.requests[i].c, spec.requests[i].c + spec.requests[i].n,
                                  KIND_V, device).cpu() for i in idx])
        pool.append(lay.block_table[idx], [spec.requests[i].c for i in idx],
                    [spec.requests[i].n for i in idx], ks, vs)
    return pool


def _group_needed(spec, g, sel):
    """Some selected request reads group g's physical prefix blocks."""
    return any(spec.shared_blocks(j) > 0 and g in [x for x, _ in spec.group_chain(spec.requests[j].group)]
               for j in sel)


def run(spec, lay=None, req_sel=None, pool=None, device="cpu"):
    """fp64 (O [T][H_q][d], LSE [T][H_q]) for the whole batch (rows of
    unselected requests are 0 / nan)."""
    lay = lay or make_layout(spec)
    pool = fill_pool(spec, lay, req_sel, pool, device)
    c = np.array([r.c for r in spec.requests], np.int32)
    n = np.array([r.n for r in spec.requests], np.int32)
    q = q_values(spec)
    if getattr(spec, "rope", None):
        pos = np.concatenate([np.arange(r.c, r.c + r.n) for r in spec.requests]) if spec.requests else []
        q = rope_bf16(q, pos, *spec.rope)
    return pool.attention(lay.block_table, c, n, q, spec.H_q, req_sel=req_sel)
