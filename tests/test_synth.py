"""The seeded generators: determinism, distribution, shapes (CPU)."""
import numpy as np
import torch

from synth.configs import make_config, make_fuzz, CONFIG_NAMES
from synth.layout import history_steps, make_layout
from synth.values import KIND_K, gen_block, kv_values


def test_values_deterministic_and_unit_scale():
    pos = torch.arange(0, 4096)
    a = gen_block(0, KIND_K, 7, pos, 8, 128)
    b = gen_block(0, KIND_K, 7, pos, 8, 128)
    assert torch.equal(a.view(torch.int16), b.view(torch.int16))
    x = a.double()
    assert abs(x.mean().item()) < 0.01 and abs(x.std().item() - 1) < 0.01
    assert x.abs().max().item() <= 2 * 3 ** 0.5 + 1e-6
    c = gen_block(1, KIND_K, 7, pos, 8, 128)
    assert not torch.equal(a, c)


def test_values_position_slices_consistent():
    spec = make_config("toy_a", 0)
    full = kv_values(spec, 1, 0, 33, KIND_K)
    part = kv_values(spec, 1, 10, 20, KIND_K)
    assert torch.equal(full[10:20], part)
    # shared-prefix content identical across group members, private part differs
    o = kv_values(spec, 2, 0, 33, KIND_K)
    assert torch.equal(full[:16], o[:16]) and not torch.equal(full[16:], o[16:])


def test_configs_shapes():
    for name in CONFIG_NAMES:
        spec = make_config(name, 0)
        assert spec.H_q % spec.H_kv == 0 and spec.T > 0
    assert make_config("c1").T == 576 and make_config("c2").T == 256 and make_config("c3").T == 768
    assert make_config("toy_a").T == 18 and make_config("toy_b").T == 18


def test_layout_covers_and_history():
    for seed in range(20):
        spec = make_fuzz(seed)
        lay = make_layout(spec)
        used = [x for x in lay.block_table.ravel() if x >= 0]
        # shared ids appear once per member, private ids exactly once
        for i, r in enumerate(spec.requests):
            nb = -(-(r.c + r.n) // spec.B)
            assert (lay.block_table[i, :nb] >= 0).all()
        assert max(used) < lay.num_blocks
        for st in history_steps(spec, lay):
            assert all(n >= 1 for n in st.n)
