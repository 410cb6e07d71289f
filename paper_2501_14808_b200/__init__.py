"""Thin Python binding of libhygen.so (include/hygen.h): argument marshalling only.

Every function keeps the C name (hg_*).  Device buffers are torch tensors
(data_ptr() is passed); host arrays are numpy.  There is no fallback: if
libhygen.so is missing, importing the binding's functions raises.  Build it
with ``python -m paper_2501_14808_b200.build`` (or __graft_entry__.build()).
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
SO_PATH = os.environ.get("HG_SO_OVERRIDE") or os.path.join(_HERE, "libhygen.so")   # override: A/B variants

HG_OK, HG_E_INVALID, HG_E_OOM, HG_E_SHARED_WRITE, HG_E_RANK_DEFICIENT, HG_E_CUDA, HG_E_NCCL, \
    HG_E_UNSUPPORTED = range(8)

HG_FEAT_S_P, HG_FEAT_S_D, HG_FEAT_S_P2, HG_FEAT_S_D2, HG_FEAT_N_P, HG_FEAT_N_D, HG_FEAT_P2, HG_FEAT_D_CTX = \
    (1 << k for k in range(8))
HG_MASK_EQ1 = HG_FEAT_S_P | HG_FEAT_S_P2 | HG_FEAT_S_D2 | HG_FEAT_N_P | HG_FEAT_N_D
HG_MASK_EQ2 = HG_FEAT_S_P | HG_FEAT_S_P2 | HG_FEAT_N_P | HG_FEAT_N_D
HG_MASK_ATTN = HG_FEAT_S_P | HG_FEAT_P2 | HG_FEAT_D_CTX | HG_FEAT_N_D | HG_FEAT_N_P
HG_FIT_RELATIVE = 1 << 8   # OR into the mask: least squares on (pred - y) / y


class HgError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"hg status {status}: {msg}")
        self.status = status


P = ctypes.c_void_p
i32 = ctypes.c_int32
i64 = ctypes.c_int64


class hg_kv_pool_desc(ctypes.Structure):
    _fields_ = [("num_blocks", i32), ("block_size", i32), ("num_kv_heads", i32), ("head_dim", i32),
                ("device", i32), ("k_cache", P), ("v_cache", P)]


class hg_batch(ctypes.Structure):
    _fields_ = [("num_reqs", i32), ("max_blocks_per_req", i32), ("block_table", P), ("cached_len", P),
                ("new_len", P), ("is_offline", P), ("shared_prefix_blocks", P)]


class hg_rope(ctypes.Structure):
    _fields_ = [("theta", ctypes.c_double), ("rotary_dim", i32)]


class hg_attn_opts(ctypes.Structure):
    _fields_ = [("split_tokens", i32), ("disable_prefix_pass", i32), ("disable_tc", i32), ("num_sms", i32),
                ("events", P * 6), ("debug_trace", P), ("rope", ctypes.POINTER(hg_rope)),
                ("disable_prefill_split", i32), ("debug_sk_trace", P), ("route", i32)]


class hg_plan_stats(ctypes.Structure):
    _fields_ = [("tc_tiles", i32), ("prefix_tiles", i32), ("splitk_items", i32), ("combine_rows", i32),
                ("kernels", i32), ("kv_bytes_unique", i64), ("kv_bytes_read", i64), ("append_mode", i32)]


class hg_features(ctypes.Structure):
    _fields_ = [(n, ctypes.c_double) for n in ("S_p", "S_d", "S_p2", "S_d2", "N_p", "N_d", "P2", "D_ctx")]

    def as_array(self):
        return np.array([getattr(self, n) for n, _ in self._fields_], np.float64)


class hg_predictor(ctypes.Structure):
    _fields_ = [("w", ctypes.c_double * 9), ("feature_mask", i32), ("n_samples", i32), ("train_mape", ctypes.c_double)]


_SIGS = {
    "hg_last_error": ([], ctypes.c_char_p),
    "hg_get_num_blocks": ([i32, i32], i32),
    "hg_kv_pool_create": ([P, P], i32),
    "hg_kv_pool_destroy": ([P], i32),
    "hg_kv_alloc": ([P, i32, P], i32),
    "hg_kv_retain": ([P, P, i32], i32),
    "hg_kv_release": ([P, P, i32], i32),
    "hg_kv_num_free": ([P], i32),
    "hg_kv_refcount": ([P, i32], i32),
    "hg_kv_append": ([P, P, P, P, P], i32),
    "hg_kv_append_rope": ([P, P, P, P, P, P], i32),
    "hg_hybrid_attention_workspace_size": ([P, P, i32, P], i32),
    "hg_hybrid_attention": ([P, P, i32, P, P, P, P, ctypes.c_size_t, P], i32),
    "hg_hybrid_attention_ex": ([P, P, i32, P, P, P, P, ctypes.c_size_t, P, P], i32),
    "hg_hybrid_step_host": ([P, P, i32, P, P, P, P, P, ctypes.c_size_t, P], i32),
    "hg_hybrid_step_host_async": ([P, P, i32, P, P, P, P, P, ctypes.c_size_t, P], i32),
    "hg_hybrid_step_host_plan": ([P, P, i32], i32),
    "hg_hybrid_step": ([P, P, i32, P, P, P, P, P, P, ctypes.c_size_t, P, P], i32),
    "hg_hybrid_step_host_workspace_size": ([P, P, i32, P], i32),
    "hg_batch_indices": ([P, P, P, P, P, P], i32),
    "hg_last_plan_stats": ([P, P], i32),
    "hg_plan_rows": ([P, i32, i32, i32, i32, i32, i32, P, P, ctypes.c_int64, P], i32),
    "hg_comm_unique_id": ([P], i32),
    "hg_comm_init": ([P, i32, i32, i32, P], i32),
    "hg_comm_destroy": ([P], i32),
    "hg_comm_window_create": ([P, ctypes.c_size_t, P, P], i32),
    "hg_comm_window_open": ([P, P], i32),
    "hg_out_proj_rs": ([P, i32, i32, i32, P, P, P, P], i32),
    "hg_hybrid_attention_tp_proj_workspace_size": ([P, P, P, i32, P], i32),
    "hg_hybrid_attention_tp_proj": ([P, P, P, i32, P, P, i32, P, P, ctypes.c_size_t, P], i32),
    "hg_hybrid_attention_tp_workspace_size": ([P, P, P, i32, P], i32),
    "hg_hybrid_attention_tp": ([P, P, P, i32, P, P, P, ctypes.c_size_t, P], i32),
    "hg_hybrid_attention_tp_ex": ([P, P, P, i32, P, P, P, ctypes.c_size_t, P, P], i32),
    "hg_hybrid_step_tp": ([P, P, P, i32, P, P, P, P, P, ctypes.c_size_t, P], i32),
    "hg_hybrid_step_tp_ex": ([P, P, P, i32, P, P, P, P, P, ctypes.c_size_t, P, P], i32),
    "hg_batch_features": ([P, i32, P], i32),
    "hg_predictor_fit": ([P, P, i32, i32, P], i32),
    "hg_predictor_predict": ([P, P], ctypes.c_double),
    "hg_slo_aware_schedule": ([P, i32, P, i32, P, i32, ctypes.c_double, i32, i32, i32, P, P, P, P, P, P], i32),
    "hg_psm_create": ([P], i32),
    "hg_psm_destroy": ([P], i32),
    "hg_psm_insert": ([P, i32, P, i32], i32),
    "hg_psm_remove": ([P, i32], i32),
    "hg_psm_size": ([P], i32),
    "hg_psm_dfs_order": ([P, P, P, i32, P], i32),
    "hg_psm_offline_schedule": ([P, i32, P, P, i32, P, i32, ctypes.c_double, i32, i32, P, P, P, P, P, P], i32),
}

_LIB = None


def lib():
    """The loaded libhygen.so.  Raises if it is missing: there is no fallback path."""
    global _LIB
    if _LIB is None:
        if not os.path.exists(SO_PATH):
            raise RuntimeError(f"{SO_PATH} missing: build it with `python -m paper_2501_14808_b200.build`")
        L = ctypes.CDLL(SO_PATH)
        for name, (args, res) in _SIGS.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = res
        _LIB = L
    return _LIB


def symbols():
    return list(_SIGS)


def _check(st: int):
    if st != HG_OK:
        raise HgError(st, lib().hg_last_error().decode())


def _ptr(x) -> Optional[int]:
    """torch tensor -> data_ptr; numpy -> address; None -> None."""
    if x is None:
        return None
    if isinstance(x, np.ndarray):
        return x.ctypes.data
    return x.data_ptr()


def _stream_ptr(stream) -> Optional[int]:
    if stream is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


def hg_get_num_blocks(tokens: int, block_size: int) -> int:
    return int(lib().hg_get_num_blocks(tokens, block_size))


class Batch:
    """Owns the host arrays behind an hg_batch (kept alive with the struct)."""

    def __init__(self, block_table, cached_len, new_len, is_offline=None, shared_prefix_blocks=None):
        self.block_table = np.ascontiguousarray(np.asarray(block_table, dtype=np.int32).reshape(len(cached_len), -1)
                                                if len(cached_len) else np.zeros((0, 1), np.int32))
        self.cached_len = np.ascontiguousarray(cached_len, dtype=np.int32)
        self.new_len = np.ascontiguousarray(new_len, dtype=np.int32)
        self.is_offline = None if is_offline is None else np.ascontiguousarray(is_offline, dtype=np.uint8)
        self.shared = None if shared_prefix_blocks is None else np.ascontiguousarray(shared_prefix_blocks, np.int32)
        self.struct = hg_batch(len(self.cached_len), self.block_table.shape[1], _ptr(self.block_table),
                               _ptr(self.cached_len), _ptr(self.new_len), _ptr(self.is_offline), _ptr(self.shared))

    @property
    def T(self) -> int:
        return int(self.new_len.sum())

    def ref(self):
        return ctypes.byref(self.struct)


class KVPool:
    """hg_kv_pool over caller-owned K/V tensors [num_blocks][H_kv][B][d] (bf16)."""

    def __init__(self, k_cache, v_cache, num_blocks: int, block_size: int, num_kv_heads: int, head_dim: int,
                 device: int = 0):
        self.k_cache, self.v_cache = k_cache, v_cache
        self.desc = hg_kv_pool_desc(num_blocks, block_size, num_kv_heads, head_dim, device,
                                    _ptr(k_cache) if not isinstance(k_cache, int) else k_cache,
                                    _ptr(v_cache) if not isinstance(v_cache, int) else v_cache)
        h = P()
        _check(lib().hg_kv_pool_create(ctypes.byref(self.desc), ctypes.byref(h)))
        self.h = h
        self.num_blocks, self.block_size, self.H_kv, self.d = num_blocks, block_size, num_kv_heads, head_dim

    def close(self):
        if self.h:
            lib().hg_kv_pool_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # allocator
    def hg_kv_alloc(self, n: int) -> np.ndarray:
        out = np.zeros(max(n, 1), np.int32)
        _check(lib().hg_kv_alloc(self.h, n, _ptr(out)))
        return out[:n]

    def hg_kv_retain(self, ids: Sequence[int]) -> None:
        a = np.ascontiguousarray(ids, np.int32)
        _check(lib().hg_kv_retain(self.h, _ptr(a), len(a)))

    def hg_kv_release(self, ids: Sequence[int]) -> None:
        a = np.ascontiguousarray(ids, np.int32)
        _check(lib().hg_kv_release(self.h, _ptr(a), len(a)))

    def hg_kv_num_free(self) -> int:
        return int(lib().hg_kv_num_free(self.h))

    def hg_kv_refcount(self, i: int) -> int:
        return int(lib().hg_kv_refcount(self.h, i))


def status_of(fn, *args) -> int:
    """Call fn and return the hg status instead of raising (error-path tests)."""
    try:
        fn(*args)
        return HG_OK
    except HgError as e:
        return e.status


def hg_kv_append(pool: KVPool, batch: Batch, k_new, v_new, stream=None) -> None:
    _check(lib().hg_kv_append(pool.h, batch.ref(), _ptr(k_new), _ptr(v_new), _stream_ptr(stream)))


def hg_kv_append_rope(pool: KVPool, batch: Batch, k_new, v_new, rope: hg_rope, stream=None) -> None:
    _check(lib().hg_kv_append_rope(pool.h, batch.ref(), _ptr(k_new), _ptr(v_new), ctypes.byref(rope),
                                   _stream_ptr(stream)))


def hg_hybrid_attention_workspace_size(pool: KVPool, batch: Batch, num_q_heads: int) -> int:
    n = ctypes.c_size_t()
    _check(lib().hg_hybrid_attention_workspace_size(pool.h, batch.ref(), num_q_heads, ctypes.byref(n)))
    return int(n.value)


def make_opts(split_tokens=0, disable_prefix_pass=False, disable_tc=False, num_sms=0, events=None,
              rope: Optional[hg_rope] = None, disable_prefill_split=False, route=0) -> hg_attn_opts:
    """events: optional 6 torch.cuda.Event(enable_timing=True) (or None entries), see hg_attn_opts.
    rope: hg_rope applied in the hg_hybrid_step prologue (kept alive by the returned struct)."""
    o = hg_attn_opts(split_tokens, int(disable_prefix_pass), int(disable_tc), num_sms)
    o.disable_prefill_split = int(disable_prefill_split)
    o.route = int(route)   # 0 automatic, 1 tcgen05 route, 2 HBM route, 3 tcgen05 prefill + split-K prefix nodes
    if rope is not None:
        o._rope_ref = rope
        o.rope = ctypes.pointer(rope)
    if events is not None:
        for k, ev in enumerate(events):
            if ev is not None:
                ev.record()   # torch creates CUDA events lazily: force creation (and mark recorded)
            o.events[k] = None if ev is None else ev.cuda_event
    return o


def hg_hybrid_attention(pool: KVPool, batch: Batch, num_q_heads: int, q, out, lse=None, workspace=None,
                        stream=None, opts: Optional[hg_attn_opts] = None) -> None:
    """out[T][H_q][d] = attention of q over the paged cache (see include/hygen.h)."""
    ws_bytes = 0 if workspace is None else workspace.numel() * workspace.element_size()
    if opts is None:
        _check(lib().hg_hybrid_attention(pool.h, batch.ref(), num_q_heads, _ptr(q), _ptr(out), _ptr(lse),
                                         _ptr(workspace), ws_bytes, _stream_ptr(stream)))
    else:
        _check(lib().hg_hybrid_attention_ex(pool.h, batch.ref(), num_q_heads, _ptr(q), _ptr(out), _ptr(lse),
                                            _ptr(workspace), ws_bytes, _stream_ptr(stream), ctypes.byref(opts)))


def hg_hybrid_step(pool: KVPool, batch: Batch, num_q_heads: int, q, k_new, v_new, out, lse=None, workspace=None,
                   stream=None, opts: Optional[hg_attn_opts] = None) -> None:
    """Fused hg_kv_append + hg_hybrid_attention (one plan, one descriptor upload)."""
    ws_bytes = 0 if workspace is None else workspace.numel() * workspace.element_size()
    _check(lib().hg_hybrid_step(pool.h, batch.ref(), num_q_heads, _ptr(q), _ptr(k_new), _ptr(v_new), _ptr(out),
                                _ptr(lse), _ptr(workspace), ws_bytes, _stream_ptr(stream),
                                None if opts is None else ctypes.byref(opts)))


def hg_hybrid_step_host_workspace_size(pool: KVPool, batch: Batch, num_q_heads: int) -> int:
    n = ctypes.c_size_t()
    _check(lib().hg_hybrid_step_host_workspace_size(pool.h, batch.ref(), num_q_heads, ctypes.byref(n)))
    return int(n.value)


def hg_hybrid_step_host(pool: KVPool, batch: Batch, num_q_heads: int, q_host, k_host, v_host, out_host,
                        workspace, stream=None) -> None:
    """End-to-end step with host buffers (pinned torch CPU tensors)."""
    _check(lib().hg_hybrid_step_host(pool.h, batch.ref(), num_q_heads, _ptr(q_host), _ptr(k_host), _ptr(v_host),
                                     _ptr(out_host), _ptr(workspace), workspace.numel() * workspace.element_size(),
                                     _stream_ptr(stream)))


def hg_hybrid_step_host_async(pool: KVPool, batch: Batch, num_q_heads: int, q_host, k_host, v_host, out_host,
                              workspace, stream=None) -> None:
    """The host step without its final synchronise (out_host valid once `stream` completes);
    uses the pool's plan-ahead for this batch if hg_hybrid_step_host_plan made one."""
    _check(lib().hg_hybrid_step_host_async(pool.h, batch.ref(), num_q_heads, _ptr(q_host), _ptr(k_host),
                                           _ptr(v_host), _ptr(out_host), _ptr(workspace),
                                           workspace.numel() * workspace.element_size(), _stream_ptr(stream)))


def hg_hybrid_step_host_plan(pool: KVPool, batch: Batch, num_q_heads: int) -> None:
    """Validate and plan `batch` for the next host step (host work only)."""
    _check(lib().hg_hybrid_step_host_plan(pool.h, batch.ref(), num_q_heads))


def hg_batch_indices(pool: KVPool, batch: Batch):
    R, T = len(batch.cached_len), batch.T
    cu = np.zeros(R + 1, np.int32)
    kv = np.zeros(max(R, 1), np.int32)
    slot = np.zeros(max(T, 1), np.int64)
    pg = np.zeros(max(R, 1), np.int32)
    _check(lib().hg_batch_indices(pool.h, batch.ref(), _ptr(cu), _ptr(kv), _ptr(slot), _ptr(pg)))
    return cu, kv[:R], slot[:T], pg[:R]


def hg_plan_rows(batch: Batch, num_q_heads: int, num_kv_heads: int, head_dim: int, num_blocks: int,
                 num_sms: int = 148, use_tc: bool = True, opts: Optional[hg_attn_opts] = None) -> np.ndarray:
    """Host-only plan inspection: int32 [n][7] rows (t, h, k0, k1, part, kind, nparts), see hygen.h."""
    n = ctypes.c_int64()
    args = (batch.ref(), num_q_heads, num_kv_heads, head_dim, num_blocks, num_sms, int(use_tc),
            None if opts is None else ctypes.byref(opts))
    _check(lib().hg_plan_rows(*args, None, 0, ctypes.byref(n)))
    out = np.zeros((n.value, 7), np.int32)
    _check(lib().hg_plan_rows(*args, _ptr(out), n.value, ctypes.byref(n)))
    return out


def hg_last_plan_stats(pool: KVPool) -> dict:
    s = hg_plan_stats()
    _check(lib().hg_last_plan_stats(pool.h, ctypes.byref(s)))
    return {n: getattr(s, n) for n, _ in s._fields_}


# ---- multi-GPU -----------------------------------------------------------------
def _preload_nccl():
    try:
        import nvidia.nccl  # noqa: F401
        path = os.path.join(os.path.dirname(nvidia.nccl.__file__), "lib", "libnccl.so.2")
        if os.path.exists(path):
            ctypes.CDLL(path, mode=ctypes.RTLD_GLOBAL)
            os.environ.setdefault("HG_NCCL_PATH", path)
    except Exception:
        pass


def hg_comm_unique_id() -> bytes:
    _preload_nccl()
    buf = (ctypes.c_char * 128)()
    _check(lib().hg_comm_unique_id(buf))
    return bytes(buf)


HG_IPC_HANDLE_BYTES = 64


class _CudaBuf:
    """Library-owned device bytes exposed through __cuda_array_interface__."""

    def __init__(self, ptr: int, nbytes: int, device: int):
        self.__cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1", "data": (ptr, False), "version": 3,
                                         "strides": None, "stream": None}


class Comm:
    """hg_comm.  uid None: no NCCL communicator (peer-window only)."""

    def __init__(self, uid: Optional[bytes], rank: int, world: int, device: int):
        buf = None
        if uid is not None:
            _preload_nccl()
            buf = (ctypes.c_char * 128).from_buffer_copy(uid)
        h = P()
        _check(lib().hg_comm_init(buf, rank, world, device, ctypes.byref(h)))
        self.h, self.rank, self.world, self.device = h, rank, world, device
        self.window_ptr = None

    def hg_comm_window_create(self, nbytes: int) -> bytes:
        """Allocates this rank's window; returns its IPC handle (to all-gather)."""
        buf = (ctypes.c_char * HG_IPC_HANDLE_BYTES)()
        ptr = P()
        _check(lib().hg_comm_window_create(self.h, nbytes, buf, ctypes.byref(ptr)))
        self.window_ptr = ptr.value
        return bytes(buf)

    def hg_comm_window_open(self, handles: Sequence[bytes]) -> None:
        blob = b"".join(handles)
        assert len(blob) == HG_IPC_HANDLE_BYTES * self.world
        buf = (ctypes.c_char * len(blob)).from_buffer_copy(blob)
        _check(lib().hg_comm_window_open(self.h, buf))

    def window(self, shape, dtype=None):
        """The gathered-output window as a torch tensor view (no copy)."""
        import torch
        dtype = dtype or torch.bfloat16
        n = int(np.prod(shape))
        holder = _CudaBuf(self.window_ptr, n * torch.empty((), dtype=dtype).element_size(), self.device)
        return torch.as_tensor(holder, device=f"cuda:{self.device}").view(dtype).view(*shape)

    def close(self):
        if self.h:
            lib().hg_comm_destroy(self.h)
            self.h = None


def hg_hybrid_attention_tp_workspace_size(pool: KVPool, comm: Comm, batch: Batch, num_q_heads_total: int) -> int:
    n = ctypes.c_size_t()
    _check(lib().hg_hybrid_attention_tp_workspace_size(pool.h, comm.h, batch.ref(), num_q_heads_total,
                                                       ctypes.byref(n)))
    return int(n.value)


def hg_hybrid_attention_tp(pool: KVPool, comm: Comm, batch: Batch, num_q_heads_total: int, q_local, out_gathered,
                           workspace, stream=None, opts: Optional[hg_attn_opts] = None) -> None:
    if opts is None:
        _check(lib().hg_hybrid_attention_tp(pool.h, comm.h, batch.ref(), num_q_heads_total, _ptr(q_local),
                                            _ptr(out_gathered), _ptr(workspace),
                                            workspace.numel() * workspace.element_size(), _stream_ptr(stream)))
    else:
        _check(lib().hg_hybrid_attention_tp_ex(pool.h, comm.h, batch.ref(), num_q_heads_total, _ptr(q_local),
                                               _ptr(out_gathered), _ptr(workspace),
                                               workspace.numel() * workspace.element_size(), _stream_ptr(stream),
                                               ctypes.byref(opts)))


def hg_hybrid_step_tp(pool: KVPool, comm: Comm, batch: Batch, num_q_heads_total: int, q_local, k_new_local,
                      v_new_local, out_gathered, workspace, stream=None, opts: Optional[hg_attn_opts] = None) -> None:
    """Fused sharded step: append of this rank's KV-head slice + hg_hybrid_attention_tp."""
    args = (pool.h, comm.h, batch.ref(), num_q_heads_total, _ptr(q_local), _ptr(k_new_local), _ptr(v_new_local),
            _ptr(out_gathered), _ptr(workspace), workspace.numel() * workspace.element_size(), _stream_ptr(stream))
    if opts is None:
        _check(lib().hg_hybrid_step_tp(*args))
    else:
        _check(lib().hg_hybrid_step_tp_ex(*args, ctypes.byref(opts)))


def hg_out_proj_rs(comm: Comm, T: int, K: int, N: int, o_local, w_local, y_shard, stream=None) -> None:
    _check(lib().hg_out_proj_rs(comm.h, T, K, N, _ptr(o_local), _ptr(w_local), _ptr(y_shard), _stream_ptr(stream)))


def hg_hybrid_attention_tp_proj_workspace_size(pool: KVPool, comm: Comm, batch: Batch, num_q_heads_total: int) -> int:
    n = ctypes.c_size_t()
    _check(lib().hg_hybrid_attention_tp_proj_workspace_size(pool.h, comm.h, batch.ref(), num_q_heads_total,
                                                            ctypes.byref(n)))
    return int(n.value)


def hg_hybrid_attention_tp_proj(pool: KVPool, comm: Comm, batch: Batch, num_q_heads_total: int, q_local, w_local,
                                N: int, y_shard, workspace, stream=None) -> None:
    _check(lib().hg_hybrid_attention_tp_proj(pool.h, comm.h, batch.ref(), num_q_heads_total, _ptr(q_local),
                                             _ptr(w_local), N, _ptr(y_shard), _ptr(workspace),
                                             workspace.numel() * workspace.element_size(), _stream_ptr(stream)))


# ---- predictor -------------------------------------------------------------------
def hg_batch_features(batch: Batch, block_size: int = 16) -> hg_features:
    f = hg_features()
    _check(lib().hg_batch_features(batch.ref(), block_size, ctypes.byref(f)))
    return f


def hg_predictor_fit(X, y_ms, feature_mask: int) -> hg_predictor:
    """X: sequence of hg_features, or a float64 array [n][8] (the same memory layout, passed zero-copy)."""
    if isinstance(X, np.ndarray):
        arr = np.ascontiguousarray(X, np.float64).reshape(-1, 8)
        ptr, n = _ptr(arr), arr.shape[0]
    else:
        arr = (hg_features * len(X))(*X)
        ptr, n = ctypes.addressof(arr), len(X)
    y = np.ascontiguousarray(y_ms, np.float64)
    m = hg_predictor()
    _check(lib().hg_predictor_fit(ptr, _ptr(y), n, feature_mask, ctypes.byref(m)))
    return m


def hg_predictor_predict(model: hg_predictor, x: hg_features) -> float:
    return float(lib().hg_predictor_predict(ctypes.byref(model), ctypes.byref(x)))


def features_from_array(a) -> hg_features:
    return hg_features(*[float(v) for v in a])


# ---- SLO-aware scheduling (Alg. 1) ------------------------------------------------
class hg_sched_req(ctypes.Structure):
    _fields_ = [("cached", i32), ("prompt_left", i32), ("shared_prefix_tokens", i32), ("group", i32)]


class hg_sched_entry(ctypes.Structure):
    _fields_ = [("index", i32), ("tokens", i32), ("t_req", ctypes.c_double)]


HG_SCHED_MAX_GROUPS = 256


class hg_sched_state(ctypes.Structure):
    """The batch under construction across the phases of one iteration (include/hygen.h)."""
    _fields_ = [("features", ctypes.c_double * 8), ("intercept_charged", i32), ("n_groups", i32),
                ("groups", i32 * HG_SCHED_MAX_GROUPS)]


def hg_slo_aware_schedule(model: hg_predictor, running, queue, latency_budget_ms: float, chunk_budget: int,
                          memory_blocks: int, phase_online: bool, block_size: int = 16, state: hg_sched_state = None):
    """running / queue: sequences of (cached, prompt_left, shared_prefix_tokens, group).
    state: hg_sched_state carried from the previous phase of the same batch (None: a batch of its own).
    Returns ([(index, tokens, t_req)], t_left, c_left, m_left)."""
    R = (hg_sched_req * max(len(running), 1))(*[hg_sched_req(*r) for r in running])
    Q = (hg_sched_req * max(len(queue), 1))(*[hg_sched_req(*r) for r in queue])
    out = (hg_sched_entry * max(len(running) + len(queue), 1))()
    n = ctypes.c_int32()
    t, c, m = ctypes.c_double(), ctypes.c_int32(), ctypes.c_int32()
    _check(lib().hg_slo_aware_schedule(ctypes.byref(model), block_size, R, len(running), Q, len(queue),
                                       latency_budget_ms, chunk_budget, memory_blocks, int(phase_online),
                                       None if state is None else ctypes.byref(state), out,
                                       ctypes.byref(n), ctypes.byref(t), ctypes.byref(c), ctypes.byref(m)))
    return [(out[k].index, out[k].tokens, out[k].t_req) for k in range(n.value)], t.value, c.value, m.value


# ---- Prefix Sharing Maximization (Alg. 3) -----------------------------------------
class PrefixTree:
    """hg_psm: prefix tree T_p over offline prompts (DFS order = PSM admission order)."""

    def __init__(self):
        h = P()
        _check(lib().hg_psm_create(ctypes.byref(h)))
        self.h = h

    def close(self):
        if self.h:
            lib().hg_psm_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def hg_psm_insert(self, request_id: int, tokens) -> None:
        a = np.ascontiguousarray(tokens, np.int32)
        _check(lib().hg_psm_insert(self.h, request_id, _ptr(a) if a.size else None, int(a.size)))

    def hg_psm_remove(self, request_id: int) -> None:
        _check(lib().hg_psm_remove(self.h, request_id))

    def hg_psm_size(self) -> int:
        return int(lib().hg_psm_size(self.h))

    def hg_psm_dfs_order(self, max_n: int = None):
        n = self.hg_psm_size() if max_n is None else max_n
        ids = np.zeros(max(n, 1), np.int32)
        lcp = np.zeros(max(n, 1), np.int32)
        k = ctypes.c_int32()
        _check(lib().hg_psm_dfs_order(self.h, _ptr(ids), _ptr(lcp), n, ctypes.byref(k)))
        return ids[:k.value].tolist(), lcp[:k.value].tolist()


def hg_psm_offline_schedule(model: hg_predictor, tree: PrefixTree, running, by_id, latency_budget_ms: float,
                            chunk_budget: int, memory_blocks: int, block_size: int = 16,
                            state: hg_sched_state = None):
    R = (hg_sched_req * max(len(running), 1))(*[hg_sched_req(*r) for r in running])
    I = (hg_sched_req * max(len(by_id), 1))(*[hg_sched_req(*r) for r in by_id])
    out = (hg_sched_entry * max(len(running) + len(by_id), 1))()
    n = ctypes.c_int32()
    t, c, m = ctypes.c_double(), ctypes.c_int32(), ctypes.c_int32()
    _check(lib().hg_psm_offline_schedule(ctypes.byref(model), block_size, tree.h, R, len(running), I, len(by_id),
                                         latency_budget_ms, chunk_budget, memory_blocks,
                                         None if state is None else ctypes.byref(state), out, ctypes.byref(n),
                                         ctypes.byref(t), ctypes.byref(c), ctypes.byref(m)))
    return [(out[k].index, out[k].tokens, out[k].t_req) for k in range(n.value)], t.value, c.value, m.value
