"""hg_slo_aware_schedule (Alg. 1, NEXT-1) against the plain mirror oracle/scheduler.py,
the worked values restated from SPEC.md, and the algorithm's invariants (CPU)."""
import numpy as np
import pytest

import paper_2501_14808_b200 as hg
from oracle import scheduler as S


def model(w):
    m = hg.hg_predictor()
    for k, v in enumerate(w):
        m.w[k] = v
    return m


def test_get_max_tokens_spec_example():
    """weights S_p 0.1, S_p^2 1e-4, N_p 0.5 (intercept 0), t = 20 ms,
    c = 4096, memory unbounded, remaining 4096: l is the largest integer with
    0.1 l + 1e-4 l^2 + 0.5 <= 20.  By hand: l = 167 (19.9889 ms; 168 gives 20.1224)."""
    w = [0, 0.1, 0, 1e-4, 0, 0.5, 0, 0, 0]
    out, t, c, m = hg.hg_slo_aware_schedule(model(w), [], [(0, 4096, 0, -1)], 20.0, 4096, 1 << 20, False)
    assert out[0][0] == 0 and out[0][1] == 167
    assert abs(out[0][2] - (16.7 + 1e-4 * 167 ** 2 + 0.5)) < 1e-9
    assert c == 4096 - 167 and m == (1 << 20) - 11   # GET_NUM_BLOCKS(167) = 11


def test_decode_marginal_spec_example():
    """empty batch, S_d weight 0.05, N_d weight 0.2, S_d^2 off -> 0.25 ms."""
    w = [0, 0, 0.05, 0, 0, 0, 0.2, 0, 0]
    out, t, _, _ = hg.hg_slo_aware_schedule(model(w), [(100, 0, 0, -1)], [], 10.0, 0, 0, False)
    assert out == [(0, 0, pytest.approx(0.25, abs=1e-12))]
    assert t == pytest.approx(9.75, abs=1e-12)


def test_budget_zero_and_intercept():
    w = [2.0, 0.1, 0, 0, 0, 0.5, 0, 0, 0]
    out, t, _, _ = hg.hg_slo_aware_schedule(model(w), [], [(0, 100, 0, -1)], 2.0, 512, 100, False)
    assert out == [] and t == pytest.approx(0.0)         # the intercept consumed the whole budget
    out, _, _, _ = hg.hg_slo_aware_schedule(model(w), [(50, 0, 0, -1)], [], 2.0, 512, 100, True)
    assert len(out) == 1                                   # online decodes are admitted regardless


def _rand_case(rng):
    nr, nq = int(rng.integers(0, 12)), int(rng.integers(0, 8))
    run = []
    for _ in range(nr):
        left = 0 if rng.random() < 0.6 else int(rng.integers(1, 3000))
        g = int(rng.integers(-1, 3))
        run.append((int(rng.integers(1, 6000)), left, 1024 if g >= 0 else 0, g))
    q = [(int(rng.integers(0, 100)), int(rng.integers(0, 4000)), 0, -1) for _ in range(nq)]
    w = np.abs(rng.standard_normal(9)) * np.array([0.05, 1e-3, 1e-3, 1e-7, 1e-4, 0.02, 0.01, 1e-7, 5e-6])
    if rng.random() < 0.3:   # non-monotone (negative) weights exercise the downward scan
        w[1] = -w[1]
    return w, run, q, float(rng.uniform(0.05, 3.0)), int(rng.integers(0, 2049)), int(rng.integers(0, 400)), \
        bool(rng.random() < 0.5)


@pytest.mark.parametrize("seed", range(300))
def test_matches_mirror(seed):
    rng = np.random.default_rng(seed)
    w, run, q, t, c, m, online = _rand_case(rng)
    got, gt, gc, gm = hg.hg_slo_aware_schedule(model(w), run, q, t, c, m, online)
    exp, et, ec, em = S.schedule(list(w), 16, run, q, t, c, m, online)
    assert [(a, b) for a, b, _ in got] == [(a, b) for a, b, _ in exp]
    np.testing.assert_allclose([x for _, _, x in got], [x for _, _, x in exp], rtol=1e-9, atol=1e-12)
    assert (gc, gm) == (ec, em) and abs(gt - et) < 1e-9


@pytest.mark.parametrize("seed", range(100))
def test_offline_budget_safety_and_additivity(seed):
    """Offline phase: every admitted entry fits, so sum t_req <= t - w0;
    marginals add up to predict(final) - predict(empty)."""
    rng = np.random.default_rng(1000 + seed)
    w, run, q, t, c, m, _ = _rand_case(rng)
    w[1] = abs(w[1])
    out, tl, _, _ = hg.hg_slo_aware_schedule(model(w), run, q, t, c, m, False)
    assert sum(x for _, _, x in out) <= t - w[0] + 1e-9
    assert tl >= -1e-9 or not out
    entries = []
    for idx, l, _ in out:
        r = run[idx] if idx < len(run) else q[idx - len(run)]
        entries.append(("d", r[0], 1, r[3], r[2]) if l == 0 else ("p", r[0], l, r[3], r[2]))
    total = S._lin(w, S._features(entries)) - S._lin(w, S._features([]))
    assert abs(sum(x for _, _, x in out) - total) < 1e-9
