"""Pins of the NEXT-row mirrors themselves (oracle/scheduler.py, oracle/psm.py),
independent of the library: the worked values SPEC.md restates from Alg. 1
(S:264 decode marginal, S:276 get_max_tokens by exhaustive scan) and the
paper's own PSM example, asserted on the mirror functions, so a
misreading shared by mirror and library cannot hide behind their agreement.
Then the two-phase batch (Alg. 2) on library and mirror alike."""
import json
import os

import numpy as np
import pytest

from oracle import psm as OP
from oracle import scheduler as S

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "psm_example.json")))
# weight vector layout: w[0] intercept, then hg_features order S_p, S_d, S_p2, S_d2, N_p, N_d, P2, D_ctx


def test_mirror_decode_marginal_spec_264():
    """empty batch, S_d weight 0.05, N_d weight 0.2, S_d^2 off -> 0.25 ms
    (one decode row adds S_d = 1 and N_d = 1: 0.05 + 0.2)."""
    w = [0, 0, 0.05, 0, 0, 0, 0.2, 0, 0]
    out, t, c, m = S.schedule(w, 16, [(100, 0, 0, -1)], [], 10.0, 0, 0, False)
    assert out == [(0, 0, pytest.approx(0.25, abs=1e-12))]
    assert t == pytest.approx(9.75, abs=1e-12)
    # and with S_d^2 on, the second decode's marginal grows by w * (2 S_d + 1)
    w2 = [0, 0, 0.05, 0, 0.01, 0, 0.2, 0, 0]
    out, _, _, _ = S.schedule(w2, 16, [(100, 0, 0, -1), (7, 0, 0, -1)], [], 10.0, 0, 0, False)
    assert out[0][2] == pytest.approx(0.25 + 0.01 * 1, abs=1e-12)
    assert out[1][2] == pytest.approx(0.25 + 0.01 * 3, abs=1e-12)


def test_mirror_get_max_tokens_spec_276():
    """weights S_p 0.1, S_p^2 1e-4, N_p 0.5, t = 20 ms, c = 4096, memory
    unbounded, 4096 left: l is the largest integer with 0.1 l + 1e-4 l^2 + 0.5 <= 20,
    found here by the exhaustive scan over [0, 4096] the spec prescribes."""
    w = [0, 0.1, 0, 1e-4, 0, 0.5, 0, 0, 0]
    scan = max(l for l in range(0, 4097) if 0.1 * l + 1e-4 * l * l + 0.5 <= 20.0)
    assert scan == 167
    out, t, c, m = S.schedule(w, 16, [], [(0, 4096, 0, -1)], 20.0, 4096, 1 << 20, False)
    assert out[0][:2] == (0, scan)
    assert out[0][2] == pytest.approx(0.1 * scan + 1e-4 * scan ** 2 + 0.5, abs=1e-12)
    assert c == 4096 - scan and m == (1 << 20) - (-(-scan // 16))   # GET_NUM_BLOCKS(167) = 11
    # budget non-binding -> l = min(c, remaining, memory cap); t = 0 -> nothing
    assert S.schedule(w, 16, [], [(0, 300, 0, -1)], 1e9, 4096, 1 << 20, False)[0][0][1] == 300
    assert S.schedule(w, 16, [], [(0, 300, 0, -1)], 1e9, 4096, 5, False)[0][0][1] == 80
    assert S.schedule(w, 16, [], [(0, 300, 0, -1)], 0.0, 4096, 1 << 20, False)[0] == []


def test_mirror_psm_paper_example_210():
    """queue (What is ML, How to code, What is AI, How to debug); PSM
    orders it (What is ML, What is AI), (How to code, How to debug)."""
    tr = OP.Trie()
    for rid, toks in enumerate(GOLD["queue"]):
        tr.insert(rid, toks)
    order, lcp = tr.lcp_with_prev()
    assert order == GOLD["psm_order"] and lcp == GOLD["lcp_with_prev"]
    assert [order[k:k + 2] for k in (0, 2)] == GOLD["psm_batches_of_two"]


def test_mirror_offline_schedule_paper_example_210():
    """Alg. 3 over the P:210 queue with a system that 'can process two offline
    requests per batch' (each prompt is 3 tokens; a chunk budget of 6 tokens admits
    exactly two): the first batch is (What is ML, What is AI), and after removing
    them the next is (How to code, How to debug)."""
    w = [0, 0.001, 0, 0, 0, 0, 0, 0, 0]
    tr = OP.Trie()
    by_id = []
    for rid, toks in enumerate(GOLD["queue"]):
        tr.insert(rid, toks)
        by_id.append((0, len(toks), 0, -1))
    batches = []
    for _ in range(2):
        out, _, _, _ = OP.offline_schedule(w, 16, tr, [], by_id, 10.0, 6, 100)
        batches.append([idx for idx, _, _ in out])
    assert batches == GOLD["psm_batches_of_two"]


def test_mirror_decode_gate_reading_r16():
    """Alg. 3's decode gate read as `t < t_req => break` (R16): a running decode that
    does not fit ends the pass, one that fits is admitted."""
    w = [0, 0, 1.0, 0, 0, 0, 0, 0, 0]
    out, t, _, _ = OP.offline_schedule(w, 16, OP.Trie(), [(10, 0, 0, -1)] * 3, [], 2.5, 0, 0)
    assert [x[0] for x in out] == [0, 1] and t == pytest.approx(0.5)


# ---- two phases on one batch (Alg. 2) -----------------------------------
def _model(w):
    import paper_2501_14808_b200 as hg
    m = hg.hg_predictor()
    for k, v in enumerate(w):
        m.w[k] = v
    return m


def test_two_phase_mirror_cross_terms():
    """The offline phase prices its chunk against the online batch: with the S_p^2
    term the marginal of l offline tokens after L online ones is
    w (2 L l + l^2), not w l^2 -- and the intercept is charged once."""
    w = [1.0, 0, 0, 1e-4, 0, 0, 0, 0, 0]
    batch = []
    on, t, c, m = S.schedule(w, 16, [], [(0, 100, 0, -1)], 10.0, 300, 1000, True, batch)
    off, t2, _, _ = S.schedule(w, 16, [], [(0, 50, 0, -1)], t, c, m, False, batch)
    assert on[0][2] == pytest.approx(1e-4 * 100 ** 2)
    assert off[0][2] == pytest.approx(1e-4 * (2 * 100 * 50 + 50 ** 2))
    assert t2 == pytest.approx(10.0 - 1.0 - 1e-4 * 150 ** 2)


@pytest.mark.parametrize("seed", range(80))
def test_two_phase_library_matches_mirror_and_sums_to_batch(seed):
    """Library (hg_sched_state) == mirror (shared batch list) over an online then an
    offline phase; w0 + the marginals of both phases == predict(whole batch) when no
    marginal is clamped (monotone weights) -- SPEC.md:282's additivity across phases."""
    import paper_2501_14808_b200 as hg
    rng = np.random.default_rng(7000 + seed)
    w = list(np.abs(rng.standard_normal(9)) * np.array([0.05, 1e-3, 1e-3, 1e-7, 1e-4, 0.02, 0.01, 1e-7, 5e-6]))

    def reqs(k):
        out = []
        for _ in range(k):
            left = 0 if rng.random() < 0.6 else int(rng.integers(1, 2000))
            g = int(rng.integers(-1, 3))
            # a member's cache holds its shared prefix: c >= 512
            out.append((int(rng.integers(512 if g >= 0 else 1, 5000)), left, 512 if g >= 0 else 0, g))
        return out
    on_run, on_q, off_run, off_q = reqs(int(rng.integers(0, 8))), reqs(int(rng.integers(0, 4))), \
        reqs(int(rng.integers(0, 8))), reqs(int(rng.integers(0, 4)))
    t, c, m = float(rng.uniform(0.2, 3.0)), int(rng.integers(0, 2048)), int(rng.integers(0, 400))
    st = hg.hg_sched_state()
    g1 = hg.hg_slo_aware_schedule(_model(w), on_run, on_q, t, c, m, True, state=st)
    g2 = hg.hg_slo_aware_schedule(_model(w), off_run, off_q, *g1[1:], False, state=st)
    batch = []
    e1 = S.schedule(w, 16, on_run, on_q, t, c, m, True, batch)
    e2 = S.schedule(w, 16, off_run, off_q, *e1[1:], False, batch)
    for got, exp in ((g1, e1), (g2, e2)):
        assert [(a, b) for a, b, _ in got[0]] == [(a, b) for a, b, _ in exp[0]]
        np.testing.assert_allclose([x for _, _, x in got[0]], [x for _, _, x in exp[0]], rtol=1e-9, atol=1e-12)
        assert got[2:] == exp[2:] and abs(got[1] - exp[1]) < 1e-9
    entries = []
    for phase, (run, q) in ((g1, (on_run, on_q)), (g2, (off_run, off_q))):
        for idx, l, _ in phase[0]:
            r = run[idx] if idx < len(run) else q[idx - len(run)]
            entries.append(("d", r[0], 1, r[3], r[2]) if l == 0 else ("p", r[0], l, r[3], r[2]))
    whole = w[0] + S._lin(w, S._features(entries))
    assert abs(w[0] + sum(x for p in (g1, g2) for _, _, x in p[0]) - whole) < 1e-9
    assert abs((t - g2[1]) - whole) < 1e-9   # the budget spent is the batch's prediction
    assert list(st.features) == pytest.approx(S._features(entries), rel=1e-12, abs=1e-12)
