"""Pins for the fp64 oracle (oracle/oracle.c) against things other than itself:
brute force on logical sequences, torch's textbook SDPA, closed forms and the
invariants the paper's batch model fixes (chunked == whole prefill, decode ==
last prefill row, shared prefix == private copies).  CPU only."""
import numpy as np
import pytest
import torch

from oracle import OraclePool, merge_partials
from oracle.brute import attention_dense
from oracle.run import fill_pool, run
from synth.configs import BatchSpec, Request, make_config, make_fuzz, make_fuzz_nested
from synth.layout import make_layout
from synth.values import KIND_K, KIND_V, kv_values, q_values


def f64(x):
    return x.to(torch.float64).numpy()


def logical_kv(spec, i):
    r = spec.requests[i]
    return (f64(kv_values(spec, i, 0, r.c + r.n, KIND_K)), f64(kv_values(spec, i, 0, r.c + r.n, KIND_V)))


def rows_of(spec, i):
    start = sum(r.n for r in spec.requests[:i])
    return slice(start, start + spec.requests[i].n)


def brute_check(spec, tol=1e-13):
    out, lse = run(spec)
    q = f64(q_values(spec))
    for i, r in enumerate(spec.requests):
        K, V = logical_kv(spec, i)
        o_ref, l_ref = attention_dense(q[rows_of(spec, i)], K, V, r.c)
        np.testing.assert_allclose(out[rows_of(spec, i)], o_ref, rtol=0, atol=tol)
        np.testing.assert_allclose(lse[rows_of(spec, i)], l_ref, rtol=0, atol=tol)


@pytest.mark.parametrize("seed", range(12))
def test_brute_force_tiny(seed):
    """d in {4, 8}, L <= 12, block size 4: paged oracle == dense brute force."""
    rng = np.random.default_rng(seed)
    d = [4, 8][seed % 2]
    H_kv = 1 + seed % 2
    G = [1, 2, 3][seed % 3]
    spec = BatchSpec(f"tiny{seed}", H_kv * G, H_kv, d, 4, seed)
    reqs = []
    for k in range(int(rng.integers(1, 5))):
        L = int(rng.integers(1, 13))
        n = int(rng.integers(1, L + 1))
        reqs.append(Request(L - n, n, bool(k % 2)))
    spec.requests = reqs
    brute_check(spec, tol=1e-14)


@pytest.mark.parametrize("name", ["toy_a", "toy_b"])
@pytest.mark.parametrize("q_scale", [1.0, 4.0])
def test_brute_force_toy(name, q_scale):
    brute_check(make_config(name, seed=0, q_scale=q_scale))


@pytest.mark.parametrize("seed", range(6))
def test_brute_force_fuzz(seed):
    brute_check(make_fuzz(seed))


@pytest.mark.parametrize("seed", range(8))
def test_brute_force_nested_prefixes(seed):
    """Prefix trie of depth <= 3 (NEXT-3): the paged oracle over physically shared
    root / child / grandchild blocks == dense brute force on each logical sequence."""
    spec = make_fuzz_nested(seed)
    lay = make_layout(spec)
    assert len(set(map(tuple, (row[:s] for row, s in zip(lay.block_table.tolist(), lay.shared) if s)))) >= 1
    brute_check(spec)


def test_sdpa_textbook_causal():
    """c = 0 single request: oracle == torch SDPA(is_causal=True) in fp64."""
    spec = BatchSpec("sdpa", 4, 2, 32, 16, 3, [Request(0, 40)])
    out, lse = run(spec)
    q = q_values(spec).to(torch.float64)          # [n][H_q][d]
    K, V = (torch.from_numpy(x) for x in logical_kv(spec, 0))
    Kx = K.repeat_interleave(2, dim=1)           # GQA h -> h // G
    Vx = V.repeat_interleave(2, dim=1)
    ref = torch.nn.functional.scaled_dot_product_attention(
        q.transpose(0, 1), Kx.transpose(0, 1), Vx.transpose(0, 1), is_causal=True).transpose(0, 1)
    np.testing.assert_allclose(out, ref.numpy(), rtol=0, atol=1e-13)


def test_sdpa_bottom_right_offset():
    """c > 0: row j sees keys <= c + j (explicit boolean mask to SDPA)."""
    spec = BatchSpec("sdpa2", 2, 2, 16, 16, 5, [Request(21, 9)])
    out, _ = run(spec)
    q = q_values(spec).to(torch.float64).transpose(0, 1)
    K, V = (torch.from_numpy(x).transpose(0, 1) for x in logical_kv(spec, 0))
    j = torch.arange(9)[:, None]
    p = torch.arange(30)[None, :]
    ref = torch.nn.functional.scaled_dot_product_attention(q, K, V, attn_mask=p <= 21 + j)
    np.testing.assert_allclose(out, ref.transpose(0, 1).numpy(), rtol=0, atol=1e-13)


def test_chunked_equals_whole_bitwise():
    """Prefill of N=70 whole vs chunks 16 + 33 + 21 (appending between chunks)."""
    whole = BatchSpec("w", 4, 2, 64, 16, 9, [Request(0, 70, cid=5)])
    o_whole, l_whole = run(whole)
    lay = make_layout(whole)
    pool = OraclePool(lay.num_blocks, 2, 16, 64)
    outs, lses = [], []
    c = 0
    for n in (16, 33, 21):
        part = BatchSpec("p", 4, 2, 64, 16, 9, [Request(c, n, cid=5)])
        pool = fill_pool(part, lay, pool=pool)
        o, l = pool.attention(lay.block_table, [c], [n], q_values(part), 4)
        outs.append(o)
        lses.append(l)
        c += n
    assert np.array_equal(np.concatenate(outs), o_whole)
    assert np.array_equal(np.concatenate(lses), l_whole)


def test_decode_equals_last_prefill_row_bitwise():
    N = 57
    whole = BatchSpec("w", 2, 2, 64, 16, 4, [Request(0, N, cid=3)])
    o_whole, _ = run(whole)
    dec = BatchSpec("d", 2, 2, 64, 16, 4, [Request(N - 1, 1, cid=3)])
    o_dec, _ = run(dec)
    assert np.array_equal(o_dec[0], o_whole[N - 1])


@pytest.mark.parametrize("seed", range(3))
def test_shared_prefix_equals_private_copies_bitwise(seed):
    spec = make_config("toy_a", seed)
    priv = spec.with_(requests=[r.__class__(**{**r.__dict__, "share": False}) for r in spec.requests])
    o_s, l_s = run(spec)
    o_p, l_p = run(priv)
    assert make_layout(spec).num_blocks != make_layout(priv).num_blocks
    assert np.array_equal(o_s, o_p) and np.array_equal(l_s, l_p)


@pytest.mark.parametrize("seed", range(4))
def test_nested_shared_prefix_equals_private_copies_bitwise(seed):
    spec = make_fuzz_nested(seed)
    priv = spec.with_(requests=[r.__class__(**{**r.__dict__, "share": False}) for r in spec.requests])
    o_s, l_s = run(spec)
    o_p, l_p = run(priv)
    assert np.array_equal(o_s, o_p, equal_nan=True) and np.array_equal(l_s, l_p, equal_nan=True)


def test_block_permutation_invariance():
    spec = make_fuzz(3)
    o1, _ = run(spec, make_layout(spec, seed=1))
    o2, _ = run(spec, make_layout(spec, seed=2))
    assert np.array_equal(o1, o2)


def test_tags_have_no_effect():
    spec = make_config("toy_b", 1)
    flipped = spec.with_(requests=[r.__class__(**{**r.__dict__, "offline": not r.offline})
                                   for r in spec.requests])
    assert np.array_equal(run(spec)[0], run(flipped)[0])


def _manual_pool(spec, Kseq, Vseq):
    """Pool whose single request holds the given logical K/V (fp32 -> bf16)."""
    lay = make_layout(spec)
    pool = OraclePool(lay.num_blocks, spec.H_kv, spec.B, spec.d)
    r = spec.requests[0]
    pool.append(lay.block_table[:1], [0], [r.c + r.n], torch.tensor(Kseq).to(torch.bfloat16),
                torch.tensor(Vseq).to(torch.bfloat16))
    return pool, lay


def test_closed_forms():
    H, d, L = 2, 16, 37
    spec = BatchSpec("cf", H, H, d, 16, 0, [Request(L - 5, 5)])
    rng = np.random.default_rng(0)
    K = rng.standard_normal((L, H, d)).astype(np.float32)
    q = q_values(spec)
    # V == constant vector => O == v
    v = rng.standard_normal(d).astype(np.float32)
    V = np.broadcast_to(v, (L, H, d)).copy()
    pool, lay = _manual_pool(spec, K, V)
    out, _ = pool.attention(lay.block_table, [L - 5], [5], q, H)
    vb = torch.tensor(v).to(torch.bfloat16).double().numpy()
    np.testing.assert_allclose(out, np.broadcast_to(vb, out.shape), rtol=1e-14, atol=1e-14)
    # Q == 0 => O == mean of the visible V rows, LSE == ln(#visible)
    V = rng.standard_normal((L, H, d)).astype(np.float32)
    pool, lay = _manual_pool(spec, K, V)
    out, lse = pool.attention(lay.block_table, [L - 5], [5], torch.zeros(5, H, d, dtype=torch.bfloat16), H)
    Vb = torch.tensor(V).to(torch.bfloat16).double().numpy()
    for j in range(5):
        np.testing.assert_allclose(out[j], Vb[:L - 5 + j + 1].mean(axis=0), rtol=1e-13, atol=1e-14)
        np.testing.assert_allclose(lse[j], np.log(L - 5 + j + 1), rtol=1e-15)
    # a single visible key => O == v_0 exactly
    one = BatchSpec("one", H, H, d, 16, 0, [Request(0, 1)])
    pool, lay = _manual_pool(one, K[:1], V[:1])
    out, _ = pool.attention(lay.block_table, [0], [1], q[:1], H)
    assert np.array_equal(out[0], Vb[0])
    # all keys identical => uniform weights => mean of V
    Kc = np.broadcast_to(K[0], (L, H, d)).copy()
    pool, lay = _manual_pool(spec, Kc, V)
    out, _ = pool.attention(lay.block_table, [L - 5], [5], q, H)
    for j in range(5):
        np.testing.assert_allclose(out[j], Vb[:L - 5 + j + 1].mean(axis=0), rtol=1e-13, atol=1e-14)


def test_gqa_equals_duplicated_mha_bitwise():
    G = 4
    gqa = BatchSpec("g", 8, 2, 32, 16, 2, [Request(19, 7), Request(40, 1)])
    o_g, _ = run(gqa)
    lay = make_layout(gqa)
    mha = OraclePool(lay.num_blocks, 8, 16, 32)
    c = [19, 40]
    n = [7, 1]
    Kf = torch.cat([kv_values(gqa, i, 0, c[i] + n[i], KIND_K) for i in range(2)]).repeat_interleave(G, 1)
    Vf = torch.cat([kv_values(gqa, i, 0, c[i] + n[i], KIND_V) for i in range(2)]).repeat_interleave(G, 1)
    mha.append(lay.block_table, [0, 0], [c[0] + n[0], c[1] + n[1]], Kf, Vf)
    o_m, _ = mha.attention(lay.block_table, c, n, q_values(gqa), 8)
    assert np.array_equal(o_g, o_m)


@pytest.mark.parametrize("cuts", [(0, 17, 64, None), (0, 5, None), (0, 100, 200, None)])
def test_split_merge_equals_unsplit(cuts):
    spec = make_config("toy_b", 2)
    spec = spec.with_(requests=spec.requests + [Request(150, 3)])
    lay = make_layout(spec)
    pool = fill_pool(spec, lay)
    c = [r.c for r in spec.requests]
    n = [r.n for r in spec.requests]
    q = q_values(spec)
    full, lse_full = pool.attention(lay.block_table, c, n, q, spec.H_q)
    parts = []
    for lo, hi in zip(cuts[:-1], cuts[1:]):
        parts.append(pool.attention(lay.block_table, c, n, q, spec.H_q, lo=lo,
                                    hi=-1 if hi is None else hi, want_partial=True))
    O, LSE = merge_partials([p[0] for p in parts], [p[1] for p in parts], [p[2] for p in parts])
    np.testing.assert_allclose(O, full, rtol=0, atol=1e-13)
    np.testing.assert_allclose(LSE, lse_full, rtol=0, atol=1e-13)


def test_sampled_selection_matches_full():
    spec = make_fuzz(5)
    full, _ = run(spec)
    sel = [0, len(spec.requests) - 1]
    part, _ = run(spec, req_sel=sel)
    for i in sel:
        assert np.array_equal(part[rows_of(spec, i)], full[rows_of(spec, i)])


# ---- RoPE (NEXT-4 prologue, reading R24) ------------------------------------------------
from oracle.rope import rope, rope_bf16   # noqa: E402


def test_rope_identity_at_position_zero():
    x = np.random.default_rng(0).standard_normal((3, 2, 64))
    assert np.array_equal(rope(x, [0, 0, 0], 1e4), x)


@pytest.mark.parametrize("rot", [0, 32])
def test_rope_keeps_pair_norms_and_tail(rot):
    rng = np.random.default_rng(1)
    x = rng.standard_normal((5, 3, 64))
    pos = rng.integers(0, 20000, 5)
    y = rope(x, pos, 5e5, rot)
    R = rot or 64
    h = R // 2
    np.testing.assert_allclose(x[..., :h] ** 2 + x[..., h:R] ** 2, y[..., :h] ** 2 + y[..., h:R] ** 2,
                               rtol=1e-12, atol=1e-12)
    assert np.array_equal(y[..., R:], x[..., R:])


def test_rope_2d_is_the_rotation_matrix():
    """R = d = 2: f_0 = 1, so position p rotates (x0, x1) by p radians."""
    rng = np.random.default_rng(2)
    x = rng.standard_normal((4, 1, 2))
    pos = np.array([0, 1, 7, 1000])
    y = rope(x, pos, 1e4)
    for k, p in enumerate(pos):
        M = np.array([[np.cos(p), -np.sin(p)], [np.sin(p), np.cos(p)]])
        np.testing.assert_allclose(y[k, 0], M @ x[k, 0], rtol=0, atol=1e-12)


def test_rope_relative_position_property():
    """q(p + s) . k(p' + s) = q(p) . k(p'): scores depend on p - p' only."""
    rng = np.random.default_rng(3)
    q, k = rng.standard_normal((1, 1, 128)), rng.standard_normal((1, 1, 128))
    for p, pp, sh in [(5, 3, 100), (4000, 17, 9000), (0, 8191, 8000)]:
        a = (rope(q, [p + sh], 5e5) * rope(k, [pp + sh], 5e5)).sum()
        b = (rope(q, [p], 5e5) * rope(k, [pp], 5e5)).sum()
        assert abs(a - b) < 1e-9 * (1 + abs(b))


def _rope_spec(spec, theta=1e4, rot=0):
    return spec.with_(rope=(theta, rot))


def brute_check_rope(spec, tol=1e-13):
    """Paged oracle with rope == dense brute force on rotated logical sequences."""
    out, lse = run(spec)
    q = q_values(spec)
    pos = np.concatenate([np.arange(r.c, r.c + r.n) for r in spec.requests])
    q = f64(rope_bf16(q, pos, *spec.rope))
    for i, r in enumerate(spec.requests):
        K = f64(rope_bf16(kv_values(spec, i, 0, r.c + r.n, KIND_K), np.arange(r.c + r.n), *spec.rope))
        V = f64(kv_values(spec, i, 0, r.c + r.n, KIND_V))
        o_ref, l_ref = attention_dense(q[rows_of(spec, i)], K, V, r.c)
        np.testing.assert_allclose(out[rows_of(spec, i)], o_ref, rtol=0, atol=tol)
        np.testing.assert_allclose(lse[rows_of(spec, i)], l_ref, rtol=0, atol=tol)


@pytest.mark.parametrize("seed", range(4))
def test_brute_force_with_rope(seed):
    brute_check_rope(_rope_spec(make_fuzz(seed), theta=[1e4, 5e5][seed % 2], rot=[0, 32][seed // 2 % 2]))


def test_brute_force_nested_with_rope():
    brute_check_rope(_rope_spec(make_fuzz_nested(2), theta=5e5))


def test_rope_chunked_equals_whole_and_decode_bitwise():
    """Positions are absolute: with rope, chunked prefill still equals the whole
    prefill and a decode equals the last prefill row, bit for bit."""
    N = 57
    whole = BatchSpec("w", 2, 2, 64, 16, 4, [Request(0, N, cid=3)], rope=(1e4, 0))
    o_whole, _ = run(whole)
    dec = BatchSpec("d", 2, 2, 64, 16, 4, [Request(N - 1, 1, cid=3)], rope=(1e4, 0))
    o_dec, _ = run(dec)
    assert np.array_equal(o_dec[0], o_whole[N - 1])
    lay = make_layout(whole)
    pool = OraclePool(lay.num_blocks, 2, 16, 64)
    outs, c = [], 0
    for n in (16, 33, 8):
        part = BatchSpec("p", 2, 2, 64, 16, 4, [Request(c, n, cid=3)], rope=(1e4, 0))
        pool = fill_pool(part, lay, pool=pool)
        q = rope_bf16(q_values(part), np.arange(c, c + n), 1e4)
        o, _ = pool.attention(lay.block_table, [c], [n], q, 2)
        outs.append(o)
        c += n
    assert np.array_equal(np.concatenate(outs), o_whole)


# ---- output projection + reduce-scatter (NEXT-4) --------------------------------------
def test_out_proj_rs_brute_force_tiny():
    from oracle.outproj import out_proj_rs, shard_rows
    rng = np.random.default_rng(5)
    G, T, N = 3, 7, 5
    Ks = [2, 3, 4]
    O = [rng.standard_normal((T, k)) for k in Ks]
    W = [rng.standard_normal((k, N)) for k in Ks]
    shards = out_proj_rs(O, W)
    for o in range(G):
        a, b = shard_rows(T, G, o)
        assert shards[o].shape == (b - a, N)
        for t in range(a, b):
            for n in range(N):
                v = 0.0
                for r in range(G):
                    for k in range(Ks[r]):
                        v += O[r][t, k] * W[r][k, n]
                assert abs(shards[o][t - a, n] - v) < 1e-12
    assert sum(shard_rows(T, G, o)[1] - shard_rows(T, G, o)[0] for o in range(G)) == T


def test_out_proj_rs_block_identity():
    from oracle.outproj import out_proj_rs
    rng = np.random.default_rng(6)
    O = [rng.standard_normal((11, 8)) for _ in range(4)]
    W = [rng.standard_normal((8, 6)) for _ in range(4)]
    full = np.concatenate(O, axis=1) @ np.concatenate(W, axis=0)
    np.testing.assert_allclose(np.concatenate(out_proj_rs(O, W)), full, rtol=1e-12, atol=1e-12)
