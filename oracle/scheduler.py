"""Plain mirror of Alg. 1 SLO_AWARE_SCHEDULE over the linear
batch-latency predictor, for checking hg_slo_aware_schedule.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Straight-line and slow on
purpose: every marginal is predict(features of B + r) - predict(features of B)
recomputed from the whole entry list, and get_max_tokens scans l downward from
its cap, so maximality holds by construction.

Readings (R19-R21): marginal clamped at 0; the intercept is charged
once before the first request; a prefill that gets no token ends the pass
(preemption is not modelled); online decodes are admitted unconditionally and
still decrement t.
"""
from __future__ import annotations


def _features(entries):
    """Batch features (order of include/hygen.h): S_p, S_d, S_p2, S_d2, N_p, N_d, P2, D_ctx.
    entries: (kind, cached, tokens, group, shared_tokens), kind 'd' or 'p'."""
    S_p = S_d = N_p = N_d = 0
    P2 = 0.0
    D = 0
    seen = set()
    for e in entries:
        if e[0] == "w0":
            continue
        kind, c, l, g, st = e
        if kind == "d":
            S_d += 1
            N_d += 1
            D += c + 1
            if g >= 0 and st > 0:
                if g in seen:
                    D -= st
                seen.add(g)
        else:
            S_p += l
            N_p += 1
            P2 += l * (c + (l + 1) / 2.0)
    return [S_p, S_d, S_p * S_p, S_d * S_d, N_p, N_d, P2, D]


def _lin(w, f):
    return sum(w[1 + k] * f[k] for k in range(8))


def _num_blocks(l, B):
    return -(-l // B) if l > 0 else 0


def schedule(w, block_size, running, queue, t, c, m, online, batch=None):
    """running/queue: lists of (cached, prompt_left, shared_prefix_tokens, group).
    Returns ([(index, tokens, t_req)], t_left, c_left, m_left).

    batch: the iteration's batch so far, a list of feature entries shared by
    the phases of Alg. 2 (the online phase, then the offline phase
    on the same batch), extended in place; the intercept is charged by the
    phase that finds it empty of charges (batch None: a batch of its own).
    The charge is recorded as a marker entry ("w0",) that _features skips."""
    if batch is None:
        batch = []
    if ("w0",) not in batch:
        t = t - w[0]
        batch.append(("w0",))
    B = batch     # feature entries of the whole batch
    out = []

    def marg(extra):
        return max(0.0, _lin(w, _features(B + [extra])) - _lin(w, _features(B)))

    for i, (ci, left, st, g) in enumerate(running):
        if left > 0:
            continue
        e = ("d", ci, 1, g, st)
        t_req = marg(e)
        if t_req <= t or online:
            t -= t_req
            B.append(e)
            out.append((i, 0, t_req))
    cand = [(k, r) for k, r in enumerate(running) if r[1] > 0] + \
           [(len(running) + k, r) for k, r in enumerate(queue)]
    for k, (ci, left, st, g) in cand:
        if left <= 0:
            continue
        hi = min(c, left, m * block_size)
        l, t_req = 0, 0.0
        for cand_l in range(hi, 0, -1):          # largest l whose marginal fits t
            tr = marg(("p", ci, cand_l, g, st))
            if tr <= t:
                l, t_req = cand_l, tr
                break
        if l > 0:
            B.append(("p", ci, l, g, st))
            t -= t_req
            c -= l
            m -= _num_blocks(l, block_size)
            out.append((k, l, t_req))
        else:
            break
    return out, t, c, m
