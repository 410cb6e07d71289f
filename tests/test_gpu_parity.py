"""GPU parity: the CUDA path (through the C ABI) against the fp64 oracle on the
same seeded inputs.  Tolerances (north_star, BASELINE.json): rel-L2 <= 5e-3
and max-abs <= 2e-2 over the output tensor; LSE within 1e-3 absolute; the
paged cache after append bit-exact; indices bit-exact (tests/test_host_lib.py).
"""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

REL_L2, MAX_ABS, LSE_ABS = 5e-3, 2e-2, 1e-3


def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@pytest.fixture(scope="module", autouse=True)
def _lib():
    _cuda()
    import paper_2501_14808_b200 as hg
    hg.lib()   # raises if the extension is missing: no fallback
    yield


def rows_of(spec, i):
    s = sum(r.n for r in spec.requests[:i])
    return slice(s, s + spec.requests[i].n)


def compare(spec, wl, req_sel=None, check_lse=True, tag=""):
    from oracle.run import run
    o_ref, lse_ref = run(spec, wl.lay, req_sel=req_sel, device="cuda")
    out = wl.out.float().cpu().double().numpy()
    lse = wl.lse.cpu().double().numpy()
    sel = range(len(spec.requests)) if req_sel is None else req_sel
    idx = np.concatenate([np.arange(rows_of(spec, i).start, rows_of(spec, i).stop) for i in sel])
    a, b = out[idx], o_ref[idx]
    rel = np.linalg.norm(a - b) / np.linalg.norm(b)
    mx = np.abs(a - b).max()
    worst = max(np.linalg.norm(out[rows_of(spec, i)] - o_ref[rows_of(spec, i)]) /
                np.linalg.norm(o_ref[rows_of(spec, i)]) for i in sel)
    # the share of max-abs that bf16 output rounding alone explains: the GPU's bf16 O
    # against the oracle rounded to bf16 (RNE), i.e. the kernel's own error
    b16 = torch.from_numpy(b).to(torch.bfloat16).double().numpy()
    mx16 = np.abs(a - b16).max()
    msg = (f"{spec.name}{tag}: rel-L2 {rel:.3e} max-abs {mx:.3e} (vs bf16(oracle) {mx16:.3e}) "
           f"worst-request rel-L2 {worst:.3e} "
           f"({'whole tensor' if req_sel is None else f'{len(sel)} requests'}, {len(idx)} rows)")
    print(msg)
    import os
    if os.environ.get("HG_PARITY_LOG"):   # evidence log (profiles/), one line per comparison
        with open(os.environ["HG_PARITY_LOG"], "a") as f:
            f.write(msg + "\n")
    assert rel <= REL_L2 and mx <= MAX_ABS, (rel, mx)
    if check_lse:
        dl = np.abs(lse[idx] - lse_ref[idx]).max()
        assert dl <= LSE_ABS, dl
    return rel, mx


def make(spec, **kw):
    from paper_2501_14808_b200.harness import Workload
    return Workload(spec, **kw)


def test_values_generator_cpu_gpu_bit_identical():
    from synth.values import gen_block
    pos = torch.arange(0, 3000)
    a = gen_block(3, 1, 77, pos, 4, 128, scale=4.0)
    b = gen_block(3, 1, 77, pos.cuda(), 4, 128, scale=4.0).cpu()
    assert torch.equal(a.view(torch.int16), b.view(torch.int16))


@pytest.mark.parametrize("name", ["toy_a", "toy_b"])
@pytest.mark.parametrize("seed", [0, 1, 2])
@pytest.mark.parametrize("q_scale", [1.0, 4.0])
def test_toy(name, seed, q_scale):
    from synth.configs import make_config
    spec = make_config(name, seed, q_scale)
    wl = make(spec)
    wl.step()
    torch.cuda.synchronize()
    compare(spec, wl)


@pytest.mark.parametrize("name", ["toy_a", "toy_b"])
def test_append_bit_exact(name):
    from oracle.run import fill_pool
    from synth.configs import make_config
    spec = make_config(name, 0)
    wl = make(spec)
    wl.append()
    torch.cuda.synchronize()
    pool = fill_pool(spec, wl.lay)
    k = wl.k_cache.cpu().view(torch.int16).numpy().view(np.uint16)
    v = wl.v_cache.cpu().view(torch.int16).numpy().view(np.uint16)
    assert np.array_equal(k, pool.K) and np.array_equal(v, pool.V)


def test_tag_flip_bit_identical():
    from synth.configs import make_config
    spec = make_config("toy_b", 1)
    wl = make(spec)
    wl.step()
    a = wl.out.clone()
    flipped = spec.with_(requests=[r.__class__(**{**r.__dict__, "offline": not r.offline}) for r in spec.requests])
    wl2 = make(flipped, lay=wl.lay)
    wl2.step()
    torch.cuda.synchronize()
    assert torch.equal(a.view(torch.int16), wl2.out.view(torch.int16))


def test_block_permutation_within_tolerance():
    from synth.configs import make_fuzz
    from synth.layout import make_layout
    spec = make_fuzz(7)
    wl1 = make(spec, lay=make_layout(spec, seed=1))
    wl2 = make(spec, lay=make_layout(spec, seed=2))
    wl1.step()
    wl2.step()
    torch.cuda.synchronize()
    a, b = wl1.out.double(), wl2.out.double()
    assert (a - b).abs().max().item() <= MAX_ABS


@pytest.mark.parametrize("seed", range(200))
def test_fuzz(seed):
    from synth.configs import make_fuzz
    spec = make_fuzz(seed)
    wl = make(spec)
    wl.step()
    torch.cuda.synchronize()
    compare(spec, wl)


@pytest.mark.parametrize("variant", ["default", "no_tc", "split64", "no_prefix", "tc_route", "hbm_route", "route3"])
@pytest.mark.parametrize("seed", range(8))
def test_plan_variants(variant, seed):
    import paper_2501_14808_b200 as hg
    from synth.configs import make_fuzz
    spec = make_fuzz(100 + seed)
    opts = {"default": None, "no_tc": hg.make_opts(disable_tc=True), "split64": hg.make_opts(split_tokens=64),
            "no_prefix": hg.make_opts(disable_prefix_pass=True), "tc_route": hg.make_opts(route=1),
            "hbm_route": hg.make_opts(route=2), "route3": hg.make_opts(route=3)}[variant]
    wl = make(spec)
    wl.append()
    wl.attention(opts)
    torch.cuda.synchronize()
    compare(spec, wl, tag=f"[{variant}]")


def test_shared_vs_private_copies():
    from synth.configs import make_config
    spec = make_config("toy_a", 2)
    priv = spec.with_(requests=[r.__class__(**{**r.__dict__, "share": False}) for r in spec.requests])
    a, b = make(spec), make(priv)
    a.step()
    b.step()
    torch.cuda.synchronize()
    assert (a.out.double() - b.out.double()).abs().max().item() <= MAX_ABS
    compare(spec, a)
    compare(priv, b)


@pytest.mark.parametrize("name", ["c1", "c1_long", "c2", "c2_g8", "c2_none", "c2_nested", "c3", "p1", "p2"])
def test_full_size_whole_tensor(name):
    """§8(c.1) acceptance at BASELINE.json's full sizes, in the launch
    configuration bench.py times (the fused step): rel-L2 over the WHOLE output
    tensor against the fp64 oracle, max-abs, LSE, and the worst single request."""
    from synth.configs import make_config
    spec = make_config(name, 0)
    wl = make(spec)
    wl.step()
    torch.cuda.synchronize()
    compare(spec, wl)
    wl.close()


def _prefill_split_spec(case):
    from synth.configs import Request
    if case == "c4_small_chunk":   # the C4 shape the predictor under-priced: 128-token chunk at c = 5600
        return _mixed(case, 32, 8, 128, [Request(5600, 128, True), Request(3000, 1), Request(4000, 1, True),
                                         Request(100, 1)])
    if case == "mha_64rows":       # 64-row items (one Q tile), G_q = 1
        return _mixed(case, 32, 32, 128, [Request(7000, 64)])
    if case == "gqa5":             # G_q = 5: items end mid-token
        return _mixed(case, 40, 8, 128, [Request(2500, 77), Request(900, 1, True)])
    if case == "d64_two_chunks":
        return _mixed(case, 32, 8, 64, [Request(3000, 200), Request(10, 1), Request(1500, 33, True)])
    if case == "short_ctx":        # c_i < 256: no cut possible for this chunk, the other one is cut
        return _mixed(case, 32, 8, 128, [Request(200, 100), Request(4096, 100)])
    raise KeyError(case)


@pytest.mark.parametrize("case", ["c4_small_chunk", "mha_64rows", "gqa5", "d64_two_chunks", "short_ctx"])
def test_prefill_key_split(case):
    """Sparse tcgen05 grid (few prefill items over long cached contexts): each
    chunk's keys are cut into ranges written as partials and merged by the
    combine kernel.  Parity with the oracle, agreement with the unsplit plan,
    and run-to-run bitwise reproducibility."""
    import paper_2501_14808_b200 as hg
    spec = _prefill_split_spec(case)
    wl = make(spec)
    wl.step()
    torch.cuda.synchronize()
    st = hg.hg_last_plan_stats(wl.pool)
    compare(spec, wl)
    a = wl.out.clone()
    wl.attention(hg.make_opts(disable_prefill_split=True))
    torch.cuda.synchronize()
    st0 = hg.hg_last_plan_stats(wl.pool)
    assert st["tc_tiles"] > st0["tc_tiles"] and st["combine_rows"] > st0["combine_rows"], (st, st0)
    assert (a.double() - wl.out.double()).abs().max().item() <= MAX_ABS
    compare(spec, wl, tag=" (unsplit)")
    wl.attention()
    torch.cuda.synchronize()
    assert torch.equal(a.view(torch.int16), wl.out.view(torch.int16))
    wl.close()


@pytest.mark.parametrize("name,q_scale", [("p1", 8.0), ("p2", 8.0), ("c1", 4.0), ("c1_long", 4.0)])
def test_peaked(name, q_scale):
    """§8(c.6) parity matrix: peaked queries (q x 4 / q x 8)."""
    from synth.configs import make_config
    spec = make_config(name, 0, q_scale)
    wl = make(spec)
    wl.step()
    torch.cuda.synchronize()
    compare(spec, wl)
    wl.close()


@pytest.mark.parametrize("name", ["c1", "c1_long", "c2"])
def test_full_size_second_seed(name):
    """§8(c.6): C1 and C2 at seed 1 as well (different lengths and block placement)."""
    from synth.configs import make_config
    spec = make_config(name, 1)
    wl = make(spec)
    wl.step()
    torch.cuda.synchronize()
    compare(spec, wl)
    wl.close()


def test_c2_shared_vs_private_full_size():
    """§8(c.6) C2 row: the all-share batch and the same batch with private prefix
    copies agree within tolerance of each other and of the oracle."""
    from synth.configs import make_config
    a = make(make_config("c2", 0))
    a.step()
    b = make(make_config("c2_private", 0))
    b.step()
    torch.cuda.synchronize()
    d = (a.out.double() - b.out.double())
    assert d.abs().max().item() <= MAX_ABS
    assert (d.norm() / b.out.double().norm()).item() <= REL_L2
    compare(a.spec, a)
    compare(b.spec, b)
    a.close()
    b.close()


def test_empty_batch():
    import paper_2501_14808_b200 as hg
    from synth.configs import BatchSpec
    spec = BatchSpec("empty", 2, 2, 64, 16, 0, [])
    wl = make(spec)
    wl.step()
    torch.cuda.synchronize()
    assert hg.hg_last_plan_stats(wl.pool)["kernels"] == 0


def test_error_leaves_outputs_untouched():
    import paper_2501_14808_b200 as hg
    from synth.configs import make_config
    spec = make_config("toy_a", 0)
    wl = make(spec)
    wl.out.fill_(7.0)
    # block S shared by r1 but private in r2: not a valid sharing (§8(b))
    bad = hg.Batch(wl.lay.block_table, [0, 32, 32], [16, 1, 1], None, [0, 1, 0])
    k_before = wl.k_cache.clone()
    st = hg.status_of(hg.hg_hybrid_attention, wl.pool, bad, spec.H_q, wl.q, wl.out, None, wl.workspace())
    assert st == hg.HG_E_INVALID
    st = hg.status_of(hg.hg_kv_append, wl.pool, hg.Batch(wl.lay.block_table[1:], [3, 32], [1, 1], None, [1, 1]),
                      wl.k_new[:2], wl.v_new[:2])
    assert st == hg.HG_E_SHARED_WRITE
    small = torch.empty(16, dtype=torch.uint8, device="cuda")
    st = hg.status_of(hg.hg_hybrid_attention, wl.pool, wl.batch, spec.H_q, wl.q, wl.out, None, small)
    assert st == hg.HG_E_INVALID
    torch.cuda.synchronize()
    assert torch.all(wl.out == 7.0) and torch.equal(k_before, wl.k_cache)


def _e2e_spec(name):
    from synth.configs import Request, make_config
    if name == "interleaved":   # prefill chunks between decodes: several row runs per wave
        return _mixed(name, 32, 8, 128, [Request(300, 200), Request(40, 1), Request(1000, 1, True),
                                         Request(0, 77), Request(129, 1), Request(64, 300, True)])
    if name == "d64_gqa5":
        return _mixed(name, 40, 8, 64, [Request(17, 1), Request(0, 130), Request(2000, 1), Request(5, 33, True)])
    if name == "c4_small_chunk":   # prefill key cuts: the chunk's rows are merged by the combine kernel
        return _prefill_split_spec(name)
    if name == "c4_219":
        from synth.trace import c4_batch
        return c4_batch(219)
    return make_config(name, 0)


@pytest.mark.parametrize("name", ["toy_a", "toy_b", "c1", "c2", "c3", "p1", "interleaved", "d64_gqa5",
                                  "c4_small_chunk", "c4_219"])
def test_e2e_host_step_matches_device_path(name):
    """hg_hybrid_step_host (host buffers, two pipelined input waves: decode rows
    then prefill-chunk rows) runs first on a fresh pool -- so its own append
    fills the cache -- and must equal hg_hybrid_step (device buffers) bit for
    bit, output and post-append cache."""
    import paper_2501_14808_b200 as hg
    spec = _e2e_spec(name)
    wl = make(spec)
    torch.cuda.synchronize()
    qh, kh, vh = (x.cpu().pin_memory() for x in (wl.q, wl.k_new, wl.v_new))
    oh = torch.full(wl.out.shape, 7.0, dtype=torch.bfloat16).pin_memory()
    ws = torch.empty(hg.hg_hybrid_step_host_workspace_size(wl.pool, wl.batch, spec.H_q), dtype=torch.uint8,
                     device="cuda")
    # with both prefill chunks and decode rows the host step puts the prefill chunks on
    # tcgen05 tiles (they consume the second input wave) and shared prefixes on split-K
    # (route 3): the same plan on the device path
    mixed = any(r.n > 1 for r in spec.requests) and any(r.n == 1 for r in spec.requests)
    for rep in range(2):   # second call: events and streams reused
        hg.hg_hybrid_step_host(wl.pool, wl.batch, spec.H_q, qh, kh, vh, oh, ws)
        k_after, v_after = wl.k_cache.clone(), wl.v_cache.clone()
        wl.step(hg.make_opts(route=3) if mixed else None)
        torch.cuda.synchronize()
        assert torch.equal(oh.view(torch.int16), wl.out.cpu().view(torch.int16)), rep
        assert torch.equal(k_after, wl.k_cache) and torch.equal(v_after, wl.v_cache), rep
    if name in ("toy_a", "toy_b", "interleaved", "c4_small_chunk", "c4_219"):
        wl.out.copy_(oh.cuda())
        compare(spec, wl, check_lse=False, tag=" (host step)")


@pytest.mark.parametrize("name", ["toy_a", "c2", "c3"])
def test_e2e_host_step_pageable_output(name):
    """With a pinned out_host the kernels store split-K's / the combine's rows into it
    directly (zero-copy result, the test above); a pageable out_host takes the copy
    path -- each equal to the device path on the same plan, bit for bit."""
    import paper_2501_14808_b200 as hg
    spec = _e2e_spec(name)
    wl = make(spec)
    torch.cuda.synchronize()
    qh, kh, vh = (x.cpu().pin_memory() for x in (wl.q, wl.k_new, wl.v_new))
    ws = torch.empty(hg.hg_hybrid_step_host_workspace_size(wl.pool, wl.batch, spec.H_q), dtype=torch.uint8,
                     device="cuda")
    mixed = any(r.n > 1 for r in spec.requests) and any(r.n == 1 for r in spec.requests)
    for pinned in (False, True):
        oh = torch.full(wl.out.shape, 7.0, dtype=torch.bfloat16)
        oh = oh.pin_memory() if pinned else oh
        hg.hg_hybrid_step_host(wl.pool, wl.batch, spec.H_q, qh, kh, vh, oh, ws)
        # a mixed batch: the host step's route 3 (its tiles consume the second input
        # wave); the appended values are the same every call, so the cache needs no reset
        wl.step(hg.make_opts(route=3) if mixed else None)
        torch.cuda.synchronize()
        assert torch.equal(oh.view(torch.int16), wl.out.cpu().view(torch.int16)), pinned


@pytest.mark.parametrize("name", ["toy_a", "c3"])
def test_e2e_host_step_plan_ahead_async(name):
    """The pipelined host step: hg_hybrid_step_host_plan for the next batch while the
    current one runs, hg_hybrid_step_host_async (no final synchronise) -- the same bits
    as the synchronous call; a plan made for another batch object is not used (that
    call plans its own), and an invalid batch fails at plan time."""
    import paper_2501_14808_b200 as hg
    spec = _e2e_spec(name)
    wl = make(spec)
    torch.cuda.synchronize()
    qh, kh, vh = (x.cpu().pin_memory() for x in (wl.q, wl.k_new, wl.v_new))
    ws = torch.empty(hg.hg_hybrid_step_host_workspace_size(wl.pool, wl.batch, spec.H_q), dtype=torch.uint8,
                     device="cuda")
    ref = torch.full(wl.out.shape, 7.0, dtype=torch.bfloat16).pin_memory()
    hg.hg_hybrid_step_host(wl.pool, wl.batch, spec.H_q, qh, kh, vh, ref, ws)
    other = hg.Batch(wl.lay.block_table, [r.c for r in spec.requests], [r.n for r in spec.requests],
                     [int(r.offline) for r in spec.requests], wl.lay.shared)   # same content, another object
    hg.hg_hybrid_step_host_plan(wl.pool, wl.batch, spec.H_q)
    for k in range(4):
        oh = torch.full(wl.out.shape, 7.0, dtype=torch.bfloat16).pin_memory()
        b = other if k == 2 else wl.batch   # k = 2: the plan-ahead is for wl.batch, not this object
        hg.hg_hybrid_step_host_async(wl.pool, b, spec.H_q, qh, kh, vh, oh, ws)
        hg.hg_hybrid_step_host_plan(wl.pool, wl.batch, spec.H_q)   # the next step's plan, beside the GPU
        torch.cuda.current_stream().synchronize()
        assert torch.equal(oh.view(torch.int16), ref.view(torch.int16)), k
    bad = hg.Batch(wl.lay.block_table, [r.c for r in spec.requests], [r.n for r in spec.requests], None,
                   [1] + [0] * (len(spec.requests) - 1))
    if name == "toy_a":   # r0 appends into a block it would share: rejected when planned
        assert hg.status_of(hg.hg_hybrid_step_host_plan, wl.pool, bad, spec.H_q) != hg.HG_OK


def test_e2e_host_step_errors_leave_outputs_untouched():
    """hg_hybrid_step_host starts the decode rows' copies before validating; an
    invalid batch must still return its status with out_host and the pool untouched."""
    import paper_2501_14808_b200 as hg
    from synth.configs import make_config
    spec = make_config("toy_a", 0)
    wl = make(spec)
    torch.cuda.synchronize()
    qh, kh, vh = (x.cpu().pin_memory() for x in (wl.q, wl.k_new, wl.v_new))
    oh = torch.full(wl.out.shape, 7.0, dtype=torch.bfloat16).pin_memory()
    ws = torch.empty(hg.hg_hybrid_step_host_workspace_size(wl.pool, wl.batch, spec.H_q), dtype=torch.uint8,
                     device="cuda")
    k_before = wl.k_cache.clone()
    bad = hg.Batch(wl.lay.block_table, [0, 32, 32], [16, 1, 1], None, [0, 1, 0])   # S shared by r1 only
    assert hg.status_of(hg.hg_hybrid_step_host, wl.pool, bad, spec.H_q, qh, kh, vh, oh, ws) == hg.HG_E_INVALID
    small = torch.empty(4096, dtype=torch.uint8, device="cuda")
    assert hg.status_of(hg.hg_hybrid_step_host, wl.pool, wl.batch, spec.H_q, qh, kh, vh, oh, small) == hg.HG_E_INVALID
    torch.cuda.synchronize()
    assert torch.all(oh == 7.0) and torch.equal(k_before, wl.k_cache)
    hg.hg_hybrid_step_host(wl.pool, wl.batch, spec.H_q, qh, kh, vh, oh, ws)   # and the next valid call works
    wl.step(hg.make_opts(route=3))   # toy_a is mixed: the host step's route 3
    torch.cuda.synchronize()
    assert torch.equal(oh.view(torch.int16), wl.out.cpu().view(torch.int16))


def test_tp_path_world1_matches_single_gpu():
    """hg_hybrid_attention_tp on a 1-rank NCCL communicator (the only GPU count
    gpurun offers): the sharded path's workspace layout + transpose kernel."""
    import paper_2501_14808_b200 as hg
    from synth.configs import make_config
    spec = make_config("toy_b", 0)
    wl = make(spec)
    wl.step()
    torch.cuda.synchronize()
    uid = hg.hg_comm_unique_id()
    comm = hg.Comm(uid, 0, 1, torch.cuda.current_device())
    out = torch.empty_like(wl.out)
    ws = torch.empty(hg.hg_hybrid_attention_tp_workspace_size(wl.pool, comm, wl.batch, spec.H_q),
                     dtype=torch.uint8, device="cuda")
    hg.hg_hybrid_attention_tp(wl.pool, comm, wl.batch, spec.H_q, wl.q, out, ws)
    torch.cuda.synchronize()
    comm.close()
    assert torch.equal(out.view(torch.int16), wl.out.view(torch.int16))


# ---- edge shapes ---------------------------------------------------------------------
def _mixed(name, H_q, H_kv, d, reqs, seed=0):
    from synth.configs import BatchSpec
    return BatchSpec(name, H_q, H_kv, d, 16, seed, reqs)


@pytest.mark.parametrize("name", ["c1_shard_g8", "c3_shard_g8"])
def test_shard_slices_full_size(name):
    """One rank's slice of 8-way KV-head sharding at full size (c1: 4 KV heads;
    C3: 1 KV head x 8 q heads, with its prefix groups), the plans bench.py's
    shard_projection times: sampled requests against the oracle."""
    from synth.configs import make_config, shard_slice
    spec = shard_slice(make_config(name.split("_")[0], 0), 8)
    wl = make(spec)
    wl.step()
    torch.cuda.synchronize()
    compare(spec, wl)
    wl.close()


def test_fused_step_more_tokens_than_param_slots():
    """T > 3968: the fused step's append falls back from the parameter-slot kernel
    to append_dev_kernel (slots derived on the device); cache bit-exact to the
    unfused append, output against the oracle."""
    from synth.configs import Request
    reqs = [Request(100, 2048), Request(50, 2040, True)] + [Request(300 + 7 * k, 1, k % 2 == 0) for k in range(20)]
    spec = _mixed("bigT", 8, 8, 64, reqs)
    assert spec.T > 3968
    wl = make(spec)
    wl.step()
    torch.cuda.synchronize()
    k_fused = wl.k_cache.clone()
    compare(spec, wl)
    wl.append()
    torch.cuda.synchronize()
    assert torch.equal(k_fused, wl.k_cache)


def test_max_context_16k():
    """Longest contexts of the configs (block table width 1088): a decode at c=16383
    and a 2048-token chunk ending at 16K."""
    from synth.configs import Request
    spec = _mixed("maxctx", 32, 8, 128, [Request(16383, 1), Request(14336, 2048, True), Request(9000, 1, True)])
    wl = make(spec)
    wl.step()
    torch.cuda.synchronize()
    compare(spec, wl)


@pytest.mark.parametrize("H_q,H_kv", [(64, 4), (12, 4), (40, 8), (16, 1), (32, 1), (64, 1), (64, 2), (48, 1)])
def test_gqa_group_sizes(H_q, H_kv):
    """G_q = 16, 3, 5, 16: split-K row stacking (16 // G tokens per item) and
    tcgen05 stacking with hl0 != 0 (G not dividing 128); G_q = 32, 64, 32, 48:
    a decode token's q heads span several 16-row split-K items."""
    from synth.configs import Request
    reqs = [Request(300, 200), Request(40, 1), Request(1000, 1, True), Request(0, 77), Request(129, 1)]
    spec = _mixed(f"gqa{H_q}x{H_kv}", H_q, H_kv, 128, reqs)
    wl = make(spec)
    wl.step()
    torch.cuda.synchronize()
    compare(spec, wl)


def test_head_dim_64_large_prefill():
    """d = 64 through the tcgen05 kernel with 256-row items (NH = 1 smem halves)."""
    from synth.configs import Request
    reqs = [Request(c, 512, k % 2 == 1) for k, c in enumerate((0, 1000, 2000, 3000))] * 2 + [Request(500, 1)]
    spec = _mixed("d64big", 32, 32, 64, reqs)
    wl = make(spec)
    wl.step()
    torch.cuda.synchronize()
    compare(spec, wl)


def test_prefix_group_with_prefill_member():
    """A shared-prefix group whose members are a prefill chunk (reads the prefix
    itself) and decodes (prefix pass + suffix split-K + combine)."""
    from synth.configs import Request
    reqs = [Request(1024 + 300, 64, True, group=0, prefix_tokens=1024)] + \
           [Request(1024 + 50 * k, 1, True, group=0, prefix_tokens=1024) for k in range(1, 40)] + \
           [Request(700, 1), Request(1024 + 7, 1, True, group=1, prefix_tokens=512),
            Request(2000, 1, True, group=1, prefix_tokens=512)]
    spec = _mixed("grp_mixed", 32, 8, 128, reqs)
    wl = make(spec)
    wl.step()
    torch.cuda.synchronize()
    assert hg_stats(wl)["prefix_tiles"] > 0
    compare(spec, wl)


def hg_stats(wl):
    import paper_2501_14808_b200 as hg
    return hg.hg_last_plan_stats(wl.pool)


def test_run_to_run_bitwise_and_fixed_split_head_sharding():
    """R17: fixed plan + fixed merge order => bitwise reproducible; with a fixed
    split (load-independent plan) a KV-head slice computes bit-identical heads."""
    import paper_2501_14808_b200 as hg
    from synth.configs import make_config
    spec = make_config("c3", 0)
    spec = spec.with_(requests=spec.requests[:1] + spec.requests[1:257:8])   # keep it quick
    opts = hg.make_opts(split_tokens=512)
    full = make(spec)
    full.append()
    full.attention(opts)
    a = full.out.clone()
    full.attention(opts)
    torch.cuda.synchronize()
    assert torch.equal(a.view(torch.int16), full.out.view(torch.int16))
    half = spec.with_(H_kv=spec.H_kv // 2, H_q=spec.H_q // 2)   # heads 0..3 / 0..31 of the same content
    sl = make(half, lay=full.lay)
    sl.append()
    sl.attention(opts)
    torch.cuda.synchronize()
    assert torch.equal(sl.out.view(torch.int16), a[:, :half.H_q].contiguous().view(torch.int16))


@pytest.mark.parametrize("name,route", [("toy_a", 0), ("c2_g8", 0), ("toy_a", 1), ("p1", 0), ("c1", 1), ("p2", 0)])
def test_fused_step_equals_append_then_attention(name, route):
    """The fused step -- HBM route: the append beside split-K, which reads the new
    keys from the inputs; tcgen05 route: the append inside the tcgen05 kernel, on
    each CTA's idle warp in the background, request by request in the order the
    tiles need them (p1, p2: the planner finds every request appended before its
    first new-key tile), else in the prologue (toy_a) -- leaves the same cache and
    output as hg_kv_append then hg_hybrid_attention, bit for bit."""
    import paper_2501_14808_b200 as hg
    from synth.configs import make_config
    spec = make_config(name, 1)
    a, b = make(spec), make(spec)
    opts = hg.make_opts(route=route) if route else None
    a.step(opts)
    mode = hg.hg_last_plan_stats(a.pool)["append_mode"]
    b.step_unfused(opts)
    torch.cuda.synchronize()
    if name in ("p1", "p2"):
        assert mode == 2, mode
    assert torch.equal(a.out.view(torch.int16), b.out.view(torch.int16))
    assert torch.equal(a.k_cache.view(torch.int16), b.k_cache.view(torch.int16))
    assert torch.equal(a.v_cache.view(torch.int16), b.v_cache.view(torch.int16))


# ---- nested prefix sharing (NEXT-3) ------------------------------------------------
def _unique_kv_bytes(spec, lay):
    """4*d*H_kv*U with U = unique KV slots of the batch: every physically shared
    block once, private positions per row."""
    shared = set()
    U = 0
    for i, r in enumerate(spec.requests):
        s = int(lay.shared[i])
        U += r.c + r.n - s * spec.B
        shared.update(int(x) for x in lay.block_table[i][:s])
    return 4 * spec.d * spec.H_kv * (U + len(shared) * spec.B)


@pytest.mark.parametrize("seed", range(60))
def test_nested_fuzz(seed):
    from synth.configs import make_fuzz_nested
    spec = make_fuzz_nested(seed)
    wl = make(spec)
    wl.step()
    torch.cuda.synchronize()
    compare(spec, wl)
    assert hg_stats(wl)["kv_bytes_unique"] == _unique_kv_bytes(spec, wl.lay)


@pytest.mark.parametrize("variant", ["no_tc", "no_prefix", "split64", "tc_route", "hbm_route", "route3"])
@pytest.mark.parametrize("seed", range(6))
def test_nested_plan_variants(variant, seed):
    import paper_2501_14808_b200 as hg
    from synth.configs import make_fuzz_nested
    spec = make_fuzz_nested(100 + seed)
    opts = {"no_tc": hg.make_opts(disable_tc=True), "split64": hg.make_opts(split_tokens=64),
            "no_prefix": hg.make_opts(disable_prefix_pass=True), "tc_route": hg.make_opts(route=1),
            "hbm_route": hg.make_opts(route=2), "route3": hg.make_opts(route=3)}[variant]
    wl = make(spec)
    wl.append()
    wl.attention(opts)
    torch.cuda.synchronize()
    compare(spec, wl, tag=f"[{variant}]")


def test_c2_nested_full_size():
    """256 decodes: a 1024-token root shared by all, 8 x 512-token children shared by
    32 each.  Two tile-map levels: the root read once for 256 members, each child
    once for its 32; the rest per request by split-K."""
    from synth.configs import make_config
    spec = make_config("c2_nested", 0)
    wl = make(spec)
    wl.step()
    torch.cuda.synchronize()
    st = hg_stats(wl)
    # HBM route (the decode pass dominates; members would re-read 40 % of the unique
    # bytes, so the nodes stay): 16-row split-K items of 4 members x G_q=4:
    # root 256 / 4 = 64 items, each child 32 / 4 = 8 -- per KV head
    assert st["prefix_tiles"] == spec.H_kv * (256 // 4 + 8 * 32 // 4), st
    assert st["kv_bytes_unique"] == _unique_kv_bytes(spec, wl.lay)
    compare(spec, wl)
    # tcgen05 route: root 256 x 4 = 1024 stacked rows; children 32 x 4 = 128 rows each;
    # beside the (much longer) split-K pass the planner takes 256-row items: H_kv*(4 + 8)
    import paper_2501_14808_b200 as hg
    wl.attention(hg.make_opts(route=1))
    torch.cuda.synchronize()
    assert hg_stats(wl)["prefix_tiles"] == spec.H_kv * (1024 // 256 + 8)
    compare(spec, wl, tag=" (tcgen05 route)")
    wl.close()


@pytest.mark.parametrize("seed", range(60))
def test_mixed_feature_fuzz(seed):
    """Everything at once on random small batches: nested prefix tries, GQA group
    sizes 1-64, d in {64, 128}, RoPE on/off, and the plan switches (fixed split,
    no prefix pass, no tcgen05), through the fused step, against the oracle."""
    import paper_2501_14808_b200 as hg
    from synth.configs import make_fuzz, make_fuzz_nested
    rng = np.random.default_rng(50_000 + seed)
    G = int(rng.choice([1, 2, 4, 8, 16, 32, 64]))
    d = int(rng.choice([64, 128]))
    spec = (make_fuzz_nested if seed % 2 else make_fuzz)(seed, G_q=G, H_kv=int(rng.choice([1, 2])), d=d)
    if rng.random() < 0.5:
        spec = spec.with_(rope=(float(rng.choice([1e4, 5e5])), int(rng.choice([0, 32]))))
    opts = [None, hg.make_opts(split_tokens=int(rng.choice([16, 64, 256]))), hg.make_opts(disable_prefix_pass=True),
            hg.make_opts(disable_tc=True)][seed % 4]
    wl = make(spec)
    wl.step(opts)
    torch.cuda.synchronize()
    compare(spec, wl, tag=f"[mixed {seed}]")
