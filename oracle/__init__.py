"""CPU oracle for the hybrid-batch attention hot path.

TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / ``--impl reference`` legs may import this package.  It shares
no code with ``paper_2501_14808_b200`` (the product) and never imports it.

Contents (each function cites the passage it follows):
  oracle.c      fp64 paged attention + append (ctypes below: OraclePool)
  brute.py      dense numpy softmax(QK^T/sqrt(d)+mask)V on logical sequences
  mirror.py     integer mirror: GET_NUM_BLOCKS, batch indices, prefix groups,
                block allocator (smallest-free-first, refcounts)
  predictor.py  Eq. 1 / Eq. 2 features, OLS fit, predict, MAPE

Parity status of each function is listed in DESIGN.md §Oracle.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None


def build(force: bool = False) -> str:
    """Compile oracle.c -> liboracle.so with gcc (-O2 -fopenmp, no fast-math)."""
    so = os.path.join(_HERE, "liboracle.so")
    src = os.path.join(_HERE, "oracle.c")
    if force or not os.path.exists(so) or os.path.getmtime(so) < os.path.getmtime(src):
        tmp = so + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-shared", "-fPIC", src, "-o", tmp, "-lm"])
        os.replace(tmp, so)
    return so


def lib():
    global _LIB
    if _LIB is None:
        L = ctypes.CDLL(build())
        P = ctypes.c_void_p
        i32, i64 = ctypes.c_int32, ctypes.c_int64
        L.oracle_append.argtypes = [P, P, i64, i32, i32, i32, i32, P, i32, P, P, P, P]
        L.oracle_append.restype = i32
        L.oracle_attention_range.argtypes = [P, P, i64, i32, i32, i32, i32, P, i32, P, P, P, i32,
                                             P, i32, i64, i64, P, P, P, P]
        L.oracle_attention_range.restype = i32
        L.oracle_num_threads.restype = i32
        L.oracle_set_num_threads.argtypes = [i32]
        L.oracle_set_num_threads.restype = None
        L.oracle_set_num_threads(len(os.sched_getaffinity(0)))   # all host cores (torchrun sets OMP_NUM_THREADS=1)
        _LIB = L
    return _LIB


def num_threads() -> int:
    return int(lib().oracle_num_threads())


def _p(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _bits(x) -> np.ndarray:
    """bf16 tensor / uint16 array -> contiguous uint16 numpy array (bit copy)."""
    if isinstance(x, np.ndarray):
        return np.ascontiguousarray(x, dtype=np.uint16)
    import torch
    return np.ascontiguousarray(x.detach().cpu().contiguous().view(torch.int16).numpy().view(np.uint16))


class OraclePool:
    """Paged KV pool [num_blocks][H_kv][B][d] of bf16 bits (uint16).

    np.zeros maps pages lazily, so a full-size pool costs memory only for the
    blocks actually written (sampled full-size checks stay cheap).
    """

    def __init__(self, num_blocks: int, H_kv: int, B: int, d: int):
        self.num_blocks, self.H_kv, self.B, self.d = num_blocks, H_kv, B, d
        self.K = np.zeros((num_blocks, H_kv, B, d), dtype=np.uint16)
        self.V = np.zeros((num_blocks, H_kv, B, d), dtype=np.uint16)

    @staticmethod
    def _table(block_table):
        bt = np.ascontiguousarray(np.asarray(block_table, dtype=np.int32))
        if bt.ndim == 1:
            bt = bt.reshape(1, -1)
        return bt

    def append(self, block_table, c, n, k_new, v_new) -> None:
        bt = self._table(block_table)
        c = np.ascontiguousarray(c, dtype=np.int32)
        n = np.ascontiguousarray(n, dtype=np.int32)
        kb, vb = _bits(k_new), _bits(v_new)
        assert kb.size == int(n.sum()) * self.H_kv * self.d
        rc = lib().oracle_append(_p(self.K), _p(self.V), self.num_blocks, self.H_kv, self.B, self.d,
                                 len(c), _p(bt), bt.shape[1], _p(c), _p(n), _p(kb), _p(vb))
        if rc != 0:
            raise ValueError("oracle_append: invalid block table")

    def attention(self, block_table, c, n, q, H_q: int, req_sel=None, lo: int = 0, hi: int = -1,
                  want_partial: bool = False):
        """fp64 attention; returns (out [T][H_q][d], lse [T][H_q]) or, with
        want_partial, (o, m, l).  Rows of unselected requests are left 0 / nan."""
        bt = self._table(block_table)
        c = np.ascontiguousarray(c, dtype=np.int32)
        n = np.ascontiguousarray(n, dtype=np.int32)
        qb = _bits(q)
        T = int(n.sum())
        assert qb.size == T * H_q * self.d
        sel = None if req_sel is None else np.ascontiguousarray(req_sel, dtype=np.int32)
        out = np.zeros((T, H_q, self.d), dtype=np.float64)
        mx = np.full((T, H_q), np.nan)
        sm = np.full((T, H_q), np.nan)
        lse = np.full((T, H_q), np.nan)
        rc = lib().oracle_attention_range(
            _p(self.K), _p(self.V), self.num_blocks, self.H_kv, self.B, self.d, len(c), _p(bt),
            bt.shape[1], _p(c), _p(n), _p(qb), H_q, _p(sel), 0 if sel is None else len(sel),
            int(lo), int(hi), _p(out), _p(mx), _p(sm), _p(lse))
        if rc != 0:
            raise ValueError("oracle_attention: invalid block table or shape")
        if want_partial:
            return out, mx, sm
        return out, lse


def merge_partials(os_, ms, ls):
    """Merge partial (o_s, m_s, l_s) triples over splits s (axis 0), SURVEY §8(a) a.7:
    M = max_s m_s;  O = sum_s e^{m_s-M} l_s o_s / sum_s e^{m_s-M} l_s;
    LSE = M + ln sum_s e^{m_s-M} l_s.  Empty splits carry m=-inf, l=0."""
    os_, ms, ls = np.asarray(os_, np.float64), np.asarray(ms, np.float64), np.asarray(ls, np.float64)
    M = np.max(ms, axis=0)
    Ms = np.where(np.isfinite(M), M, 0.0)
    a = np.where(np.isfinite(ms), np.exp(ms - Ms[None]), 0.0) * ls
    den = a.sum(axis=0)
    O = (a[..., None] * os_).sum(axis=0) / den[..., None]
    return O, Ms + np.log(den)
