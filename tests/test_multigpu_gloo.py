"""Multi-GPU host logic on CPU: world size 2 over gloo.

Rank r owns KV heads [r*H_kv/G, (r+1)*H_kv/G) and their q heads; block tables
are replicated (the allocator is deterministic); outputs are all-gathered
rank-major and transposed to [T][H_q][d].  The oracle per shard, gathered,
must equal the unsharded oracle bit-for-bit (fp64, same arithmetic per head),
and the library allocator must make identical decisions on every rank.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _shard_spec(spec, rank, world):
    """The rank's slice: same requests, H_kv/G KV heads and H_q/G q heads."""
    return spec.with_(H_kv=spec.H_kv // world, H_q=spec.H_q // world)


def _worker(rank, world, port, name, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import OraclePool
        from synth.configs import make_config, make_fuzz
        from synth.layout import history_steps, make_layout
        from synth.values import KIND_K, KIND_V, kv_values, q_values
        import paper_2501_14808_b200 as hg

        spec = make_config(name, 0) if not name.startswith("fuzz") else make_fuzz(int(name[4:]), H_kv=2, G_q=4)
        lay = make_layout(spec)
        Hk, Hq = spec.H_kv // world, spec.H_q // world
        # replicated, deterministic allocation: every rank gets the same ids
        pool = hg.KVPool(1 << 20, 1 << 20, 64, 16, Hk, spec.d)
        ids = pool.hg_kv_alloc(7)
        pool.hg_kv_release(ids[2:4])
        ids2 = pool.hg_kv_alloc(3)
        mine = torch.tensor(np.concatenate([ids, ids2]).astype(np.int64))
        allids = [torch.zeros_like(mine) for _ in range(world)]
        dist.all_gather(allids, mine)
        # the rank's KV heads / q heads of the same logical batch
        kh = slice(rank * Hk, (rank + 1) * Hk)
        qh = slice(rank * Hq, (rank + 1) * Hq)
        op = OraclePool(lay.num_blocks, Hk, spec.B, spec.d)
        for st in history_steps(spec, lay):
            ks = torch.cat([kv_values(spec, i, c, c + n, KIND_K)[:, kh] for i, c, n in zip(st.req, st.c, st.n)])
            vs = torch.cat([kv_values(spec, i, c, c + n, KIND_V)[:, kh] for i, c, n in zip(st.req, st.c, st.n)])
            op.append(st.tables, st.c, st.n, ks, vs)
        c = [r.c for r in spec.requests]
        n = [r.n for r in spec.requests]
        ks = torch.cat([kv_values(spec, i, r.c, r.c + r.n, KIND_K)[:, kh] for i, r in enumerate(spec.requests)])
        vs = torch.cat([kv_values(spec, i, r.c, r.c + r.n, KIND_V)[:, kh] for i, r in enumerate(spec.requests)])
        op.append(lay.block_table, c, n, ks, vs)
        out, lse = op.attention(lay.block_table, c, n, q_values(spec)[:, qh].contiguous(), Hq)
        local = torch.from_numpy(out)                         # [T][Hq/G][d]
        gathered = [torch.zeros_like(local) for _ in range(world)]
        dist.all_gather(gathered, local)                      # rank-major [G][T][Hl][d]
        full = torch.stack(gathered, 1).reshape(local.shape[0], spec.H_q, spec.d)   # -> [T][G*Hl][d]
        if rank == 0:
            q.put((full.numpy(), [a.numpy().tolist() for a in allids]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name", ["toy_a", "fuzz3", "fuzz11"])
def test_head_sharded_gather_equals_unsharded(name):
    from oracle.run import run
    from synth.configs import make_config, make_fuzz
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, name, q)) for r in range(world)]
    for p in procs:
        p.start()
    full, allids = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    spec = make_config(name, 0) if not name.startswith("fuzz") else make_fuzz(int(name[4:]), H_kv=2, G_q=4)
    ref, _ = run(spec)
    assert np.array_equal(full, ref)
    assert all(a == allids[0] for a in allids)


def test_gather_transpose_layout_mirror():
    """[G][T][Hl*d] rank-major NCCL layout -> [T][G][Hl*d]: the transpose the
    library's gather_transpose_kernel performs, restated in numpy."""
    G, T, E = 4, 5, 24
    src = np.arange(G * T * E).reshape(G, T, E)
    dst = np.transpose(src, (1, 0, 2))
    for t in range(T):
        for r in range(G):
            assert np.array_equal(dst[t, r], src[r, t])
