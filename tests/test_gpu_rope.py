"""NEXT-4 prologue: append + RoPE fused into hg_hybrid_step (include/hygen.h
hg_rope), against the oracle with the same rotation (oracle/rope.py, R24).
Tolerances as tests/test_gpu_parity.py."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _lib():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2501_14808_b200 as hg
    hg.lib()
    yield


def _run(spec, req_sel=None):
    from test_gpu_parity import compare, make
    wl = make(spec)
    wl.step()
    torch.cuda.synchronize()
    compare(spec, wl, req_sel=req_sel, tag="[rope]")
    return wl


@pytest.mark.parametrize("name", ["toy_a", "toy_b"])
@pytest.mark.parametrize("theta", [1e4, 5e5])
def test_toy_rope(name, theta):
    from synth.configs import make_config
    _run(make_config(name, 0).with_(rope=(theta, 0)))


@pytest.mark.parametrize("seed", range(24))
def test_fuzz_rope(seed):
    from synth.configs import make_fuzz, make_fuzz_nested
    spec = (make_fuzz_nested if seed % 3 == 2 else make_fuzz)(seed)
    rot = 32 if seed % 4 == 1 else 0
    _run(spec.with_(rope=([1e4, 5e5][seed % 2], rot)))


@pytest.mark.parametrize("name", ["c1", "c1_long", "c2_nested"])
def test_full_size_rope_whole_tensor(name):
    """Full-size configs with the rope prologue: the whole output tensor against the oracle."""
    from synth.configs import make_config
    spec = make_config(name, 0).with_(rope=(5e5 if name == "c2_nested" else 1e4, 0))
    wl = _run(spec)
    wl.close()


def test_rope_keys_in_cache_match_oracle_rotation():
    """The cached K rows after the rope prologue: within one bf16 ulp of the fp64
    rotation rounded to bf16 (fp32 rotation on the GPU), most of them identical."""
    from oracle.rope import rope_bf16
    from synth.configs import make_config
    from synth.values import KIND_K, kv_values
    from test_gpu_parity import make
    spec = make_config("toy_b", 0).with_(rope=(1e4, 0))
    wl = make(spec)
    wl.step()
    torch.cuda.synchronize()
    B = spec.B
    for i, r in enumerate(spec.requests):
        k_ref = rope_bf16(kv_values(spec, i, 0, r.c + r.n, KIND_K), np.arange(r.c + r.n), 1e4)
        rows = []
        for p in range(r.c + r.n):
            blk = int(wl.lay.block_table[i][p // B])
            rows.append(wl.k_cache[blk, :, p % B].cpu())
        got = torch.stack(rows)
        diff = (got.view(torch.int16).int() - k_ref.view(torch.int16).int()).abs()
        assert diff.max().item() <= 1
        assert (diff == 0).float().mean().item() > 0.95


def test_rope_errors():
    import paper_2501_14808_b200 as hg
    from synth.configs import make_config
    from test_gpu_parity import make
    spec = make_config("toy_a", 0)
    wl = make(spec)
    bad = [hg.hg_rope(0.0, 0), hg.hg_rope(1e4, 24), hg.hg_rope(1e4, 128)]   # theta, R % 16, R > d (d = 64)
    for r in bad:
        o = hg.make_opts(rope=r)
        with pytest.raises(hg.HgError) as e:
            hg.hg_hybrid_step(wl.pool, wl.batch, spec.H_q, wl.q, wl.k_new, wl.v_new, wl.out, wl.lse,
                              wl.workspace(), None, o)
        assert e.value.status == hg.HG_E_INVALID
    with pytest.raises(hg.HgError) as e:   # rope belongs to the step prologue only
        wl.attention(hg.make_opts(rope=hg.hg_rope(1e4, 0)))
    assert e.value.status == hg.HG_E_INVALID
    with pytest.raises(hg.HgError) as e:
        hg.hg_kv_append_rope(wl.pool, wl.batch, wl.k_new, wl.v_new, hg.hg_rope(1e4, 20))
    assert e.value.status == hg.HG_E_INVALID
