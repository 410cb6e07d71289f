"""The work plan on the host (no GPU): every query row's key ranges must tile
[0, c_i + j + 1) exactly once across the plan's items -- prefill tiles (with the
key cuts of long chunks on a sparse grid), shared-prefix node tiles (the a.4 tile
map over prefix tries) and split-K items -- with partial indices 0..n-1 when a
row is merged from n ranges and -1 when it is written directly.  Integer work:
checked exactly, through hg_plan_rows (include/hygen.h)."""
import numpy as np
import pytest

import paper_2501_14808_b200 as hg
from synth.configs import BatchSpec, CONFIG_NAMES, Request, make_config, make_fuzz, make_fuzz_nested
from synth.layout import make_layout


def _batch(spec, lay):
    return hg.Batch(lay.block_table, [r.c for r in spec.requests], [r.n for r in spec.requests],
                    [int(r.offline) for r in spec.requests], lay.shared)


def check_plan(spec, lay, num_sms=148, use_tc=True, opts=None):
    rows = hg.hg_plan_rows(_batch(spec, lay), spec.H_q, spec.H_kv, spec.d, lay.num_blocks, num_sms, use_tc, opts)
    T, H = spec.T, spec.H_q
    lim = np.concatenate([np.arange(r.c + 1, r.c + r.n + 1) for r in spec.requests]).astype(np.int64)
    t, h, k0, k1, part, kind, nparts = (rows[:, i].astype(np.int64) for i in range(7))
    assert np.all(k0 % 16 == 0), "range start not block aligned"
    key = t * H + h
    # ranges per row, empty ones included: a split-K piece past an early row's
    # causal limit (prefill rows on split-K) is an empty partial, weight 0 in the merge
    o = np.lexsort((k0, key))
    kall = key[o]
    fa = np.r_[True, kall[1:] != kall[:-1]]
    cnt_all = np.diff(np.r_[np.flatnonzero(fa), len(kall)])
    ranges = np.empty(len(key), np.int64)
    ranges[o] = np.repeat(cnt_all, cnt_all)
    ne = k1 > k0
    assert np.all(kind[~ne] == 2), "empty range outside split-K"
    kk, a0, a1, tt = key[ne], k0[ne], k1[ne], t[ne]
    o = np.lexsort((a0, kk))
    kk, a0, a1, tt = kk[o], a0[o], a1[o], tt[o]
    assert np.array_equal(np.unique(kk), np.arange(T * H)), "a row without work"
    first = np.r_[True, kk[1:] != kk[:-1]]
    last = np.r_[kk[1:] != kk[:-1], True]
    assert np.all(a0[first] == 0), "range does not start at key 0"
    assert np.all(a1[last] == lim[tt[last]]), "range does not end at the causal limit"
    assert np.all(a0[~first] == a1[np.flatnonzero(~first) - 1]), "gap or overlap between ranges"
    assert np.all(nparts == ranges), "nparts != ranges of the row"
    assert np.all(part[ranges == 1] == -1), "single-range row not written directly"
    multi = ranges > 1
    if multi.any():   # partial indices 0..n-1, each once per row
        s = np.lexsort((part[multi], key[multi]))
        pm, km = part[multi][s], key[multi][s]
        f = np.r_[True, km[1:] != km[:-1]]
        idx = np.arange(len(pm)) - np.maximum.accumulate(np.where(f, np.arange(len(pm)), 0))
        assert np.array_equal(pm, idx), "partial indices not 0..n-1"
    return rows


@pytest.mark.parametrize("name", [n for n in CONFIG_NAMES if n != "c4"])
def test_named_configs(name):
    spec = make_config(name, 0)
    check_plan(spec, make_layout(spec, seed=0))


@pytest.mark.parametrize("seed", range(40))
@pytest.mark.parametrize("num_sms", [148, 24])
def test_fuzz(seed, num_sms):
    spec = make_fuzz(seed)
    check_plan(spec, make_layout(spec, seed=seed), num_sms=num_sms)


@pytest.mark.parametrize("seed", range(40))
def test_fuzz_nested_tries(seed):
    spec = make_fuzz_nested(seed)
    check_plan(spec, make_layout(spec, seed=seed))


@pytest.mark.parametrize("opts", [dict(disable_prefix_pass=True), dict(split_tokens=256), dict(disable_tc=True),
                                  dict(disable_prefill_split=True)])
def test_plan_switches(opts):
    for seed in range(10):
        spec = make_fuzz_nested(seed)
        check_plan(spec, make_layout(spec, seed=seed), opts=hg.make_opts(**opts))


def _long(name, H_q, H_kv, d, reqs):
    return BatchSpec(name, H_q, H_kv, d, 16, 0, reqs)


LONG = {
    "c4_small_chunk": (32, 8, 128, [Request(5600, 128, True), Request(3000, 1), Request(4000, 1, True), Request(100, 1)]),
    "mha_64rows": (32, 32, 128, [Request(7000, 64)]),
    "gqa5": (40, 8, 128, [Request(2500, 77), Request(900, 1, True)]),
    "two_chunks_d64": (32, 8, 64, [Request(3000, 200), Request(10, 1), Request(1500, 33, True)]),
    "short_ctx": (32, 8, 128, [Request(200, 100), Request(4096, 100)]),
    "max_ctx": (32, 8, 128, [Request(16000, 256), Request(12000, 1)]),
}


@pytest.mark.parametrize("case", sorted(LONG))
@pytest.mark.parametrize("num_sms", [148, 40])
def test_prefill_key_cuts(case, num_sms):
    """Small chunks at long contexts: the plan cuts their keys at 128-key tile
    boundaries inside the cached prefix, and still tiles every row exactly."""
    H_q, H_kv, d, reqs = LONG[case]
    spec = _long(case, H_q, H_kv, d, reqs)
    rows = check_plan(spec, make_layout(spec, seed=1), num_sms=num_sms)
    pre = (rows[:, 5] == 0) & (rows[:, 4] >= 0)
    if num_sms == 148 and case != "short_ctx":
        assert pre.any(), "no key cut on a sparse grid"
    cuts = rows[pre]
    inner = cuts[:, 2] > 0
    assert np.all(cuts[inner, 2] % 128 == 0)
    off = hg.hg_plan_rows(_batch(spec, make_layout(spec, seed=1)), H_q, H_kv, d, make_layout(spec, seed=1).num_blocks,
                          num_sms, True, hg.make_opts(disable_prefill_split=True))
    assert not ((off[:, 5] == 0) & (off[:, 4] >= 0)).any()


def test_prefill_cuts_off_under_fixed_split():
    """split_tokens > 0 promises a load-independent plan (R17): no key cuts."""
    H_q, H_kv, d, reqs = LONG["c4_small_chunk"]
    spec = _long("c4_small_chunk", H_q, H_kv, d, reqs)
    lay = make_layout(spec, seed=1)
    rows = check_plan(spec, lay, opts=hg.make_opts(split_tokens=512))
    assert not ((rows[:, 5] == 0) & (rows[:, 4] >= 0)).any()


def test_prefill_cuts_stay_off_beside_a_large_decode_pass():
    """c1_long: a 512-token chunk at 3584 beside 64 decodes of 1-4K keys -- the
    decode pass is the long pole, so the chunk stays whole."""
    spec = make_config("c1_long", 0)
    rows = check_plan(spec, make_layout(spec, seed=0))
    assert not ((rows[:, 5] == 0) & (rows[:, 4] >= 0)).any()


def test_invalid_batch_rejected():
    spec = make_config("toy_a", 0)
    lay = make_layout(spec, seed=0)
    bad = hg.Batch(lay.block_table, [0, 32, 32], [16, 1, 1], None, [0, 1, 0])
    with pytest.raises(hg.HgError) as e:
        hg.hg_plan_rows(bad, spec.H_q, spec.H_kv, spec.d, lay.num_blocks)
    assert e.value.status == hg.HG_E_INVALID


def test_c4_batch_with_a_small_chunk_at_10k():
    """C4 batch #219 (synth.trace.c4_batch(219)): a 49-token chunk at c = 10240
    beside a 975-token chunk at c = 0 and 59 decodes.  Whole, its 8 items walk 81
    KV tiles each while everything else is done (0.222 ms); cut, 0.112 ms."""
    from synth.trace import c4_batch
    spec = c4_batch(219)
    lay = make_layout(spec, seed=219)
    rows = check_plan(spec, lay)
    cut = (rows[:, 5] == 0) & (rows[:, 4] >= 0)
    t_long = sum(r.n for r in spec.requests[:[i for i, r in enumerate(spec.requests) if r.c == 10240][0]])
    assert cut.any() and np.all(rows[cut, 0] >= t_long) and np.all(rows[cut, 0] < t_long + 49)


@pytest.mark.parametrize("G_q,H_kv", [(32, 1), (64, 1), (32, 2), (48, 1), (24, 2)])
@pytest.mark.parametrize("seed", range(6))
def test_gqa_groups_above_16(G_q, H_kv, seed):
    """G_q > 16 (MQA-like groups, P:63 batches any model's rows): a decode row's q
    heads exceed one 16-row split-K item, so each token's rows are cut into
    ceil(G_q / 16) items; every (token, q head) must still be covered exactly."""
    for make in (make_fuzz, make_fuzz_nested):
        spec = make(seed, G_q=G_q, H_kv=H_kv)
        lay = make_layout(spec, seed=seed)
        check_plan(spec, lay)
        check_plan(spec, lay, opts=hg.make_opts(disable_tc=True))
        check_plan(spec, lay, opts=hg.make_opts(split_tokens=64))


def test_decode_row_ending_inside_a_shared_block():
    """Plain hg_hybrid_attention accepts a decode row whose context ends inside a
    shared block (c_i + 1 < s_i * B; only an append forbids it).  The prefix node's
    tiles give every member the node's whole key range, so such a row may join a
    node only over the blocks it sees completely; the keys past its causal limit
    must not be covered (check_plan: ranges end exactly at c_i + 1)."""
    spec = BatchSpec("inside_shared", 8, 2, 64, 16, 0,
                     [Request(30, 1, True), Request(100, 1, True), Request(47, 1, True), Request(12, 1, True)])
    # rows 0-3 share blocks [5, 6, 7] (48 tokens) in their first columns
    bt = np.full((4, 8), -1, np.int32)
    bt[0, :2] = [5, 6]
    bt[1, :7] = [5, 6, 7, 10, 11, 12, 13]
    bt[2, :3] = [5, 6, 7]
    bt[3, :1] = [5]
    shared = [2, 3, 3, 1]
    b = hg.Batch(bt, [r.c for r in spec.requests], [1] * 4, None, shared)
    for opts in (None, hg.make_opts(split_tokens=16)):
        rows = hg.hg_plan_rows(b, spec.H_q, spec.H_kv, spec.d, 32, 148, True, opts)
        t, k1 = rows[:, 0], rows[:, 3]
        for i, r in enumerate(spec.requests):
            assert k1[t == i].max() == r.c + 1, (i, k1[t == i].max())
        # row 1 (c = 100) and row 2 (c = 47) still read blocks 5..7 once through a node
        assert (np.isin(rows[:, 5], (1, 3)) & (t == 1)).any()


@pytest.mark.parametrize("route", [1, 2, 3])
@pytest.mark.parametrize("seed", range(20))
def test_routes_tile_exactly(route, seed):
    """Both routes (tcgen05 tiles, or everything on split-K with prefix nodes as
    stacked-row split-K items) tile every row's keys exactly once."""
    for make in (make_fuzz, make_fuzz_nested):
        spec = make(seed)
        lay = make_layout(spec, seed=seed)
        rows = check_plan(spec, lay, opts=hg.make_opts(route=route))
        kinds = set(np.unique(rows[:, 5]).tolist())
        assert kinds <= {1: {0, 1, 2}, 2: {2, 3}, 3: ({0, 2, 3} if spec.H_q // spec.H_kv <= 16 else {0, 1, 2})}[route]


@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c2_nested"])
def test_auto_route_takes_hbm_route_beside_a_large_decode_pass(name):
    """The decode-dominated configs run on the HBM route (no tcgen05 items); on that
    route a shared prefix is read once per 16-row node item where its re-reads would
    be a large share of the bytes (c2_nested), else the members re-read it (L2)."""
    spec = make_config(name, 0)
    rows = check_plan(spec, make_layout(spec, seed=0))
    assert not np.isin(rows[:, 5], (0, 1)).any()
    # prefix nodes only where the members would re-read > 25 % of the unique KV bytes
    assert (rows[:, 5] == 3).any() == (name == "c2_nested")


@pytest.mark.parametrize("name", ["p1", "p2"])
def test_auto_route_keeps_tcgen05_for_prefill_heavy(name):
    spec = make_config(name, 0)
    rows = check_plan(spec, make_layout(spec, seed=0))
    assert (rows[:, 5] == 0).any()
