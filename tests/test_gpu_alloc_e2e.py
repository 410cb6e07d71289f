"""The allocator in the real flow (SURVEY §8(a) a.2 feeding a.3-a.7): block tables
built through hg_kv_alloc / hg_kv_retain on a churned pool (P:161
GET_NUM_BLOCKS, P:142 memory counted in blocks), the history and the
iteration appended through those tables, the hybrid step checked against the
fp64 oracle on the same tables, then every reference released and the pool's
conservation checked (free + live blocks = N at every point; all free
at the end)."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _spec():
    from synth.configs import BatchSpec, Request
    reqs = [Request(300, 200, False)]                                                   # online prefill chunk
    reqs += [Request(1024 + 37 * k, 1, True, group=0, prefix_tokens=1024) for k in range(24)]   # 64-block prefix
    reqs += [Request(512 + 91 * k, 1, True, group=1, prefix_tokens=512) for k in range(9)]     # 32-block prefix
    reqs += [Request(1500 + 13 * k, 1, False) for k in range(8)]                        # online decodes
    reqs += [Request(512 + 40, 33, True, group=1, prefix_tokens=512)]                   # a prefilling member
    return BatchSpec("alloc_e2e", 32, 8, 128, 16, 3, reqs)


def _num_blocks(tokens, B=16):
    import paper_2501_14808_b200 as hg
    return hg.hg_get_num_blocks(tokens, B)


def test_allocator_tables_end_to_end():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2501_14808_b200 as hg
    from oracle.run import run
    from paper_2501_14808_b200.harness import Workload
    from synth.layout import Layout, make_layout
    spec = _spec()
    B = spec.B
    N = make_layout(spec).num_blocks + 512
    wl = Workload(spec, lay=make_layout(spec, num_blocks=N), populate=False)   # only sizes the pool
    pool = wl.pool
    assert pool.hg_kv_num_free() == N
    rng = np.random.default_rng(11)
    # churn: allocate in random chunks, release a random half, so ids come back fragmented
    held = [pool.hg_kv_alloc(int(rng.integers(1, 40))) for _ in range(20)]
    for k in rng.permutation(len(held))[: len(held) // 2]:
        pool.hg_kv_release(held[k])
        held[k] = np.zeros(0, np.int32)
    churn = np.concatenate(held)

    def conserved(live_refs):
        live = set(int(x) for x in churn) | set(live_refs)
        assert pool.hg_kv_num_free() + len(live) == N

    # group prefixes: allocated once (the group's own reference), retained by each member
    gblocks = {0: pool.hg_kv_alloc(_num_blocks(1024)), 1: pool.hg_kv_alloc(_num_blocks(512))}
    W = max(_num_blocks(r.c + r.n) for r in spec.requests)
    bt = np.full((len(spec.requests), W), -1, np.int32)
    shared = np.zeros(len(spec.requests), np.int32)
    for i, r in enumerate(spec.requests):
        s = spec.shared_blocks(i)
        row = []
        if s:
            pool.hg_kv_retain(gblocks[r.group][:s])
            row += list(gblocks[r.group][:s])
        row += list(pool.hg_kv_alloc(_num_blocks(r.c + r.n) - s))   # GET_NUM_BLOCKS(l) for the rest
        bt[i, :len(row)] = row
        shared[i] = s
    live = [int(x) for x in bt[bt >= 0]] + [int(x) for g in gblocks.values() for x in g]
    conserved(live)
    for g, ids in gblocks.items():
        members = sum(1 for i, r in enumerate(spec.requests) if r.group == g and spec.shared_blocks(i))
        assert all(pool.hg_kv_refcount(int(b)) == 1 + members for b in ids)
    lay = Layout(N, bt, shared, {g: [int(x) for x in ids] for g, ids in gblocks.items()})
    wl.lay = lay
    wl.batch = hg.Batch(bt, [r.c for r in spec.requests], [r.n for r in spec.requests],
                        [int(r.offline) for r in spec.requests], shared)
    wl.populate()
    wl.step()
    torch.cuda.synchronize()
    o_ref, lse_ref = run(spec, lay, device="cuda")
    out = wl.out.double().cpu().numpy()
    rel = np.linalg.norm(out - o_ref) / np.linalg.norm(o_ref)
    mx = np.abs(out - o_ref).max()
    assert rel <= 5e-3 and mx <= 2e-2, (rel, mx)
    assert np.abs(wl.lse.double().cpu().numpy() - lse_ref).max() <= 1e-3
    assert hg.hg_last_plan_stats(pool)["prefix_tiles"] > 0   # the shared blocks went through the tile map
    # release: every request drops its row (shared blocks once per member), then the groups theirs
    for i in rng.permutation(len(spec.requests)):
        row = bt[i][bt[i] >= 0]
        pool.hg_kv_release(row)
    for ids in gblocks.values():
        assert all(pool.hg_kv_refcount(int(b)) == 1 for b in ids)
        pool.hg_kv_release(ids)
    conserved([])
    pool.hg_kv_release(churn)
    assert pool.hg_kv_num_free() == N
    assert all(pool.hg_kv_refcount(b) == 0 for b in range(N))
    wl.close()
