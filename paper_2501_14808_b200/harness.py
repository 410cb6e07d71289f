"""Load a synthetic workload (synth.BatchSpec) into a device KV pool through the
C ABI, and run the iteration.  Used by tests/ (GPU parity) and bench.py.

Everything numeric happens in libhygen.so: the history is written with
hg_kv_append, the iteration with hg_kv_append + hg_hybrid_attention.  Token
values come from synth's counter-based generator evaluated on the device.
"""
from __future__ import annotations

import ctypes
import numpy as np
import torch

import paper_2501_14808_b200 as hg
from synth.layout import Layout, history_steps, make_layout
from synth.values import KIND_K, KIND_V, kv_values, q_values


class Workload:
    def __init__(self, spec, lay: Layout = None, device="cuda", populate=True, append_chunk_tokens=1 << 16,
                 gen_device=None):
        """gen_device: where synth's generator runs (bit-identical on CPU and CUDA);
        "cpu" makes the inputs with one host-to-device copy per tensor instead of
        ~20 elementwise kernels each (smoke(): few launches besides the library's)."""
        self.spec = spec
        self.lay = lay or make_layout(spec)
        self.device = torch.device(device)
        self.gen = torch.device(gen_device) if gen_device is not None else self.device
        N, H, d = self.lay.num_blocks, spec.H_kv, spec.d
        self.k_cache = torch.zeros((N, H, spec.B, d), dtype=torch.bfloat16, device=self.device)
        self.v_cache = torch.zeros((N, H, spec.B, d), dtype=torch.bfloat16, device=self.device)
        self.pool = hg.KVPool(self.k_cache, self.v_cache, N, spec.B, H, d,
                              self.device.index if self.device.index is not None else torch.cuda.current_device())
        c = [r.c for r in spec.requests]
        n = [r.n for r in spec.requests]
        self.batch = hg.Batch(self.lay.block_table, c, n, [int(r.offline) for r in spec.requests], self.lay.shared)
        self.q = q_values(spec, device=self.gen).to(self.device)
        self.k_new = self._kv_new(KIND_K)
        self.v_new = self._kv_new(KIND_V)
        T = spec.T
        self.out = torch.empty((T, spec.H_q, d), dtype=torch.bfloat16, device=self.device)
        self.lse = torch.empty((T, spec.H_q), dtype=torch.float32, device=self.device)
        self.ws = None
        self.chunk = append_chunk_tokens
        if populate:
            self.populate()

    def _kv_new(self, kind):
        parts = [kv_values(self.spec, i, r.c, r.c + r.n, kind, device=self.gen)
                 for i, r in enumerate(self.spec.requests)]
        if not parts:
            return torch.empty((0, self.spec.H_kv, self.spec.d), dtype=torch.bfloat16, device=self.device)
        return torch.cat(parts).to(self.device)

    def populate(self):
        """History appends: every request's first c_i tokens (group prefixes once)."""
        spec = self.spec
        for st in history_steps(spec, self.lay):
            rows = list(range(len(st.c)))
            start = 0
            while start < len(rows):
                tok, end = 0, start
                while end < len(rows) and (end == start or tok + st.n[rows[end]] <= self.chunk):
                    tok += st.n[rows[end]]
                    end += 1
                sel = rows[start:end]
                ks = torch.cat([kv_values(spec, st.req[k], st.c[k], st.c[k] + st.n[k], KIND_K, device=self.gen)
                                for k in sel]).to(self.device)
                vs = torch.cat([kv_values(spec, st.req[k], st.c[k], st.c[k] + st.n[k], KIND_V, device=self.gen)
                                for k in sel]).to(self.device)
                # rows list the blocks before their write position that are shared
                shared = [st.shared[k] for k in sel]
                b = hg.Batch(np.array([st.tables[k] for k in sel], np.int32), [st.c[k] for k in sel],
                             [st.n[k] for k in sel], None, shared)
                if spec.rope:   # cached keys were appended rotated (NEXT-4 prologue)
                    hg.hg_kv_append_rope(self.pool, b, ks, vs, self.rope())
                else:
                    hg.hg_kv_append(self.pool, b, ks, vs)
                start = end
        torch.cuda.synchronize(self.device)

    def workspace(self, opts=None):
        """Workspace sized once per workload (plans with test opts may need a few
        more partial slots: 2x headroom; a too-small workspace is a loud HG_E_INVALID)."""
        if self.ws is None:
            need = hg.hg_hybrid_attention_workspace_size(self.pool, self.batch, self.spec.H_q)
            self.ws = torch.empty(max(need * 2, need + (64 << 20)), dtype=torch.uint8, device=self.device)
        return self.ws

    def append(self, stream=None):
        hg.hg_kv_append(self.pool, self.batch, self.k_new, self.v_new, stream)

    def attention(self, opts=None, lse=True, stream=None):
        hg.hg_hybrid_attention(self.pool, self.batch, self.spec.H_q, self.q, self.out,
                               self.lse if lse else None, self.workspace(opts), stream, opts)

    def rope(self):
        return hg.hg_rope(float(self.spec.rope[0]), int(self.spec.rope[1])) if self.spec.rope else None

    def step(self, opts=None, stream=None):
        """One serving iteration: fused append (+ RoPE prologue when spec.rope) + attention (hg_hybrid_step)."""
        if self.spec.rope:
            opts = opts or hg.make_opts()
            opts._rope_ref = self.rope()
            opts.rope = ctypes.pointer(opts._rope_ref)
        hg.hg_hybrid_step(self.pool, self.batch, self.spec.H_q, self.q, self.k_new, self.v_new, self.out, self.lse,
                          self.workspace(opts), stream, opts)

    def step_unfused(self, opts=None, stream=None):
        self.append(stream)
        self.attention(opts, stream=stream)

    def close(self):
        self.pool.close()
