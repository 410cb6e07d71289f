// comm.cpp -- multi-GPU step of the hot path:
// rank r owns KV heads [r*H_kv/G, (r+1)*H_kv/G) and their q-heads, runs the
// single-GPU path on its slice, then the outputs are all-gathered over NVLink
// with NCCL (tensor-parallel attention; the paper runs TP=2).
//
// NCCL is loaded with dlopen (libnccl.so.2, the copy torch ships) so the
// library has no link-time NCCL dependency; only the ABI below is used.
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <cstring>

#include "hg_internal.h"

namespace {
typedef int nccl_result;
typedef void *nccl_comm;
struct nccl_uid { char internal[128]; };
enum { kNcclBf16 = 9 };

struct NcclApi {
    bool loaded = false;
    nccl_result (*GetUniqueId)(nccl_uid *) = nullptr;
    nccl_result (*CommInitRank)(nccl_comm *, int, nccl_uid, int) = nullptr;
    nccl_result (*CommDestroy)(nccl_comm) = nullptr;
    nccl_result (*AllGather)(const void *, void *, size_t, int, nccl_comm, cudaStream_t) = nullptr;
    const char *(*GetErrorString)(nccl_result) = nullptr;
};
NcclApi g_nccl;

bool load_nccl() {
    if (g_nccl.loaded) return true;
    void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
        const char *p = getenv("HG_NCCL_PATH");
        if (p) h = dlopen(p, RTLD_NOW | RTLD_GLOBAL);
    }
    if (!h) return false;
    g_nccl.GetUniqueId = (decltype(g_nccl.GetUniqueId))dlsym(h, "ncclGetUniqueId");
    g_nccl.CommInitRank = (decltype(g_nccl.CommInitRank))dlsym(h, "ncclCommInitRank");
    g_nccl.CommDestroy = (decltype(g_nccl.CommDestroy))dlsym(h, "ncclCommDestroy");
    g_nccl.AllGather = (decltype(g_nccl.AllGather))dlsym(h, "ncclAllGather");
    g_nccl.GetErrorString = (decltype(g_nccl.GetErrorString))dlsym(h, "ncclGetErrorString");
    g_nccl.loaded = g_nccl.GetUniqueId && g_nccl.CommInitRank && g_nccl.CommDestroy && g_nccl.AllGather;
    return g_nccl.loaded;
}
}  // namespace

// Peer window: [flags: kMaxOuts x u64, padded to kWinHdr][data].  Every rank
// maps every other rank's window through CUDA IPC (NVLink peer memory).
constexpr size_t kWinHdr = 4096;

struct hg_comm {
    nccl_comm comm = nullptr;   // NULL: peer-window-only communicator
    int rank = 0, world = 1, device = 0;
    uint8_t *win = nullptr;     // this rank's window (cudaMalloc, library-owned)
    size_t win_bytes = 0;       // data bytes
    uint8_t *peer[hg::kMaxOuts] = {};   // window bases of every rank (self = win)
    bool open = false;
    unsigned long long epoch = 0;
};

using namespace hg;

namespace hg {
hg_status launch_out_proj(const uint16_t *o, const uint16_t *w, int M, int N, int K, int G, int rank, int rows_max,
                          uint16_t *const *dst, void *stream);
hg_status launch_rs_reduce(const uint16_t *recv, uint16_t *y, int rows, int rows_max, int N, int G, void *stream);
hg_status launch_gather_transpose(const uint16_t *src, uint16_t *dst, int G, int T, int row_elems, void *stream);
int pool_num_kv_heads(const hg_kv_pool *p);
int pool_head_dim(const hg_kv_pool *p);
}  // namespace hg

extern "C" hg_status hg_comm_unique_id(void *out) {
    if (!out) return fail(HG_E_INVALID, "NULL argument");
    if (!load_nccl()) return fail(HG_E_NCCL, "libnccl.so.2 not loadable (set HG_NCCL_PATH)");
    nccl_uid id;
    nccl_result r = g_nccl.GetUniqueId(&id);
    if (r) return fail(HG_E_NCCL, "ncclGetUniqueId: %d", r);
    memcpy(out, id.internal, 128);
    return HG_OK;
}

extern "C" hg_status hg_comm_init(const void *uid, int32_t rank, int32_t world, int32_t device, hg_comm **out) {
    if (!out || world < 1 || rank < 0 || rank >= world) return fail(HG_E_INVALID, "bad arguments");
    if (world > kMaxOuts) return fail(HG_E_INVALID, "world %d > %d", world, kMaxOuts);
    if (uid && !load_nccl()) return fail(HG_E_NCCL, "libnccl.so.2 not loadable (set HG_NCCL_PATH)");
    if (cudaSetDevice(device) != cudaSuccess) return fail(HG_E_CUDA, "cudaSetDevice(%d)", device);
    hg_comm *c = new hg_comm();
    if (uid) {
        nccl_uid id;
        memcpy(id.internal, uid, 128);
        nccl_result r = g_nccl.CommInitRank(&c->comm, world, id, rank);
        if (r) {
            delete c;
            return fail(HG_E_NCCL, "ncclCommInitRank: %s", g_nccl.GetErrorString ? g_nccl.GetErrorString(r) : "?");
        }
    }
    c->rank = rank;
    c->world = world;
    c->device = device;
    *out = c;
    return HG_OK;
}

extern "C" hg_status hg_comm_destroy(hg_comm *c) {
    if (!c) return HG_OK;
    if (c->comm && g_nccl.loaded) g_nccl.CommDestroy(c->comm);
    cudaSetDevice(c->device);
    for (int k = 0; k < c->world; ++k)
        if (c->peer[k] && c->peer[k] != c->win) cudaIpcCloseMemHandle(c->peer[k]);
    if (c->win) cudaFree(c->win);
    cudaGetLastError();
    delete c;
    return HG_OK;
}

extern "C" hg_status hg_comm_window_create(hg_comm *c, size_t bytes, void *ipc_handle_out, void **window_out) {
    if (!c || !ipc_handle_out || !window_out || bytes == 0) return fail(HG_E_INVALID, "bad arguments");
    if (c->win) return fail(HG_E_INVALID, "window already created");
    if (cudaSetDevice(c->device) != cudaSuccess) return fail(HG_E_CUDA, "cudaSetDevice(%d)", c->device);
    const size_t total = kWinHdr + (bytes + 255) / 256 * 256;
    if (cudaMalloc(&c->win, total) != cudaSuccess) {
        cudaGetLastError();
        c->win = nullptr;
        return fail(HG_E_OOM, "window of %zu bytes", total);
    }
    cudaIpcMemHandle_t h;
    if (cudaMemset(c->win, 0, kWinHdr) != cudaSuccess || cudaIpcGetMemHandle(&h, c->win) != cudaSuccess ||
        cudaDeviceSynchronize() != cudaSuccess) {
        cudaError_t e = cudaGetLastError();
        cudaFree(c->win);
        c->win = nullptr;
        return fail(HG_E_CUDA, "window setup: %s", cudaGetErrorString(e));
    }
    static_assert(sizeof(cudaIpcMemHandle_t) == HG_IPC_HANDLE_BYTES, "IPC handle size");
    memcpy(ipc_handle_out, &h, sizeof h);
    c->win_bytes = bytes;
    *window_out = c->win + kWinHdr;
    return HG_OK;
}

extern "C" hg_status hg_comm_window_open(hg_comm *c, const void *handles) {
    if (!c || !handles) return fail(HG_E_INVALID, "bad arguments");
    if (!c->win) return fail(HG_E_INVALID, "hg_comm_window_create first");
    if (c->open) return fail(HG_E_INVALID, "window already open");
    if (cudaSetDevice(c->device) != cudaSuccess) return fail(HG_E_CUDA, "cudaSetDevice(%d)", c->device);
    for (int k = 0; k < c->world; ++k) {
        if (k == c->rank) {
            c->peer[k] = c->win;
            continue;
        }
        cudaIpcMemHandle_t h;
        memcpy(&h, (const uint8_t *)handles + (size_t)k * HG_IPC_HANDLE_BYTES, sizeof h);
        void *ptr = nullptr;
        cudaError_t e = cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess);
        if (e != cudaSuccess) {
            cudaGetLastError();
            for (int j = 0; j < k; ++j)
                if (c->peer[j] && c->peer[j] != c->win) cudaIpcCloseMemHandle(c->peer[j]);
            memset(c->peer, 0, sizeof c->peer);
            return fail(HG_E_CUDA, "cudaIpcOpenMemHandle(rank %d): %s", k, cudaGetErrorString(e));
        }
        c->peer[k] = (uint8_t *)ptr;
    }
    c->open = true;
    return HG_OK;
}

static size_t al256(size_t x) { return (x + 255) / 256 * 256; }

extern "C" hg_status hg_hybrid_attention_tp_workspace_size(const hg_kv_pool *pool, const hg_comm *comm,
                                                           const hg_batch *batch, int32_t H_q, size_t *bytes) {
    if (!pool || !comm || !batch || !bytes) return fail(HG_E_INVALID, "NULL argument");
    if (H_q % comm->world) return fail(HG_E_INVALID, "num_q_heads %d not divisible by world %d", H_q, comm->world);
    size_t attn = 0;
    hg_status s = hg_hybrid_attention_workspace_size(pool, batch, H_q / comm->world, &attn);
    if (s) return s;
    int64_t T = 0;
    for (int i = 0; i < batch->num_reqs; ++i) T += batch->new_len[i];
    *bytes = al256(attn) + al256((size_t)T * H_q * pool_head_dim(pool) * 2);
    return HG_OK;
}

// Shared body of hg_hybrid_attention_tp / hg_hybrid_step_tp: one validated plan
// per call; k_new != NULL fuses the append (this rank's KV-head slice).
static hg_status tp_call(hg_kv_pool *pool, hg_comm *comm, const hg_batch *batch, int32_t H_q, const void *q_local,
                         const void *k_new, const void *v_new, void *out_gathered, void *workspace,
                         size_t workspace_bytes, void *stream, const hg_attn_opts *o = nullptr) {
    if (!pool || !comm || !batch) return fail(HG_E_INVALID, "NULL argument");
    if (H_q % comm->world) return fail(HG_E_INVALID, "num_q_heads %d not divisible by world %d", H_q, comm->world);
    const int G = comm->world, Hl = H_q / G, d = pool_head_dim(pool);
    size_t attn = 0;
    hg_status s = plan_attention(pool, batch, Hl, k_new != nullptr, &attn, o);
    if (s) return s;
    int64_t T = 0;
    for (int i = 0; i < batch->num_reqs; ++i) T += batch->new_len[i];
    const size_t need = al256(attn) + al256((size_t)T * H_q * d * 2);
    if (!workspace || workspace_bytes < need) return fail(HG_E_INVALID, "workspace too small (%zu < %zu)", workspace_bytes, need);
    const size_t out_bytes = (size_t)T * H_q * d * 2;
    if (comm->open && out_bytes <= comm->win_bytes) {
        // v2: every epilogue stores its O rows into all ranks' windows, at this
        // rank's head offset of the gathered [T][H_q][d] layout.  Entry barrier:
        // no rank overwrites a window its owner may still read from the last call.
        if (T == 0) return HG_OK;
        unsigned long long *fl[kMaxOuts];
        for (int k = 0; k < G; ++k) fl[k] = (unsigned long long *)comm->peer[k];
        unsigned long long *mine = (unsigned long long *)comm->win;
        OutSpec os;
        os.n = G;
        os.ld = (int64_t)H_q * d;
        for (int k = 0; k < G; ++k) os.ptr[k] = (uint16_t *)(comm->peer[k] + kWinHdr) + (size_t)comm->rank * Hl * d;
        if (k_new) {   // fused step: the entry barrier rides in the append kernel (no extra launch)
            for (int k = 0; k < G; ++k) os.bar_flags[k] = fl[k];
            os.bar_mine = mine;
            os.bar_rank = comm->rank;
            os.bar_world = G;
            os.bar_epoch = ++comm->epoch;
            os.exit_epoch = ++comm->epoch;   // the call may run the exit barrier in its last kernel
        } else {
            s = launch_peer_barrier(fl, mine, comm->rank, G, ++comm->epoch, stream);
            if (s) return s;
        }
        s = attention_planned(pool, batch, Hl, q_local, k_new, v_new, nullptr, &os, workspace, attn, stream, o);
        if (s) return s;
        // exit barrier, resident behind the attention's last kernel (PDL); on the
        // sharded HBM route it also waits for the append's device count (that append
        // ran on a side stream without a stream join, so no event wait breaks the
        // programmatic-dependent chain)
        if (!os.exit_folded) {
            const unsigned long long ep = os.exit_epoch ? os.exit_epoch : ++comm->epoch;
            s = launch_peer_barrier(fl, mine, comm->rank, G, ep, stream, true, os.wait_cnt, os.wait_target);
            if (s) return s;
        }
        uint8_t *data = comm->win + kWinHdr;
        if (out_gathered != data) {
            cudaError_t e = cudaMemcpyAsync(out_gathered, data, out_bytes, cudaMemcpyDeviceToDevice,
                                            (cudaStream_t)stream);
            if (e != cudaSuccess) return fail(HG_E_CUDA, "window copy: %s", cudaGetErrorString(e));
        }
        return HG_OK;
    }
    if (!comm->comm && G > 1) return fail(HG_E_INVALID, "no NCCL communicator and no open window of %zu bytes",
                                          out_bytes);
    uint8_t *w = (uint8_t *)workspace;
    uint16_t *gather = (uint16_t *)(w + al256(attn));  // [G][T][Hl][d], rank-major (NCCL layout)
    const size_t count = (size_t)T * Hl * d;
    uint16_t *mine = gather + (size_t)comm->rank * count;
    if (T == 0) return HG_OK;
    s = attention_planned(pool, batch, Hl, q_local, k_new, v_new, mine, nullptr, workspace, attn, stream, o);
    if (s) return s;
    if (G > 1) {
        nccl_result r = g_nccl.AllGather(mine, gather, count, kNcclBf16, comm->comm, (cudaStream_t)stream);
        if (r) return fail(HG_E_NCCL, "ncclAllGather: %s", g_nccl.GetErrorString ? g_nccl.GetErrorString(r) : "?");
    }
    // [G][T][Hl*d] -> [T][G*Hl*d]
    return launch_gather_transpose(gather, (uint16_t *)out_gathered, G, (int)T, Hl * d, stream);
}

extern "C" hg_status hg_hybrid_attention_tp(hg_kv_pool *pool, hg_comm *comm, const hg_batch *batch, int32_t H_q,
                                            const void *q_local, void *out_gathered, void *workspace,
                                            size_t workspace_bytes, void *stream) {
    return tp_call(pool, comm, batch, H_q, q_local, nullptr, nullptr, out_gathered, workspace, workspace_bytes,
                   stream);
}

extern "C" hg_status hg_hybrid_attention_tp_ex(hg_kv_pool *pool, hg_comm *comm, const hg_batch *batch, int32_t H_q,
                                               const void *q_local, void *out_gathered, void *workspace,
                                               size_t workspace_bytes, void *stream, const hg_attn_opts *opts) {
    return tp_call(pool, comm, batch, H_q, q_local, nullptr, nullptr, out_gathered, workspace, workspace_bytes,
                   stream, opts);
}

extern "C" hg_status hg_hybrid_step_tp(hg_kv_pool *pool, hg_comm *comm, const hg_batch *batch, int32_t H_q,
                                       const void *q_local, const void *k_new_local, const void *v_new_local,
                                       void *out_gathered, void *workspace, size_t workspace_bytes, void *stream) {
    if (!k_new_local || !v_new_local) return fail(HG_E_INVALID, "k_new / v_new NULL");
    return tp_call(pool, comm, batch, H_q, q_local, k_new_local, v_new_local, out_gathered, workspace,
                   workspace_bytes, stream);
}

extern "C" hg_status hg_hybrid_step_tp_ex(hg_kv_pool *pool, hg_comm *comm, const hg_batch *batch, int32_t H_q,
                                          const void *q_local, const void *k_new_local, const void *v_new_local,
                                          void *out_gathered, void *workspace, size_t workspace_bytes, void *stream,
                                          const hg_attn_opts *opts) {
    if (!k_new_local || !v_new_local) return fail(HG_E_INVALID, "k_new / v_new NULL");
    if (opts && opts->rope) return fail(HG_E_INVALID, "the sharded step has no rope prologue");
    return tp_call(pool, comm, batch, H_q, q_local, k_new_local, v_new_local, out_gathered, workspace,
                   workspace_bytes, stream, opts);
}

// ---------------------------------------------------------------------------
// NEXT-4: TP-native epilogue -- output projection + reduce-scatter (gemm.cu)
// ---------------------------------------------------------------------------
extern "C" hg_status hg_out_proj_rs(hg_comm *comm, int32_t T, int32_t K, int32_t N, const void *o_local,
                                    const void *w_local, void *y_shard, void *stream) {
    if (!comm || T < 0 || K <= 0 || N <= 0) return fail(HG_E_INVALID, "bad arguments");
    if (K % 64 || N % 128)
        return fail(HG_E_UNSUPPORTED, "out-proj: K %d must be a multiple of 64 and N %d of 128", K, N);
    if (T == 0) return HG_OK;
    if (!o_local || !w_local || !y_shard) return fail(HG_E_INVALID, "NULL buffer");
    const int G = comm->world;
    if (cudaSetDevice(comm->device) != cudaSuccess) return fail(HG_E_CUDA, "cudaSetDevice(%d)", comm->device);
    if (G == 1) {
        uint16_t *dst[1] = {(uint16_t *)y_shard};
        return launch_out_proj((const uint16_t *)o_local, (const uint16_t *)w_local, T, N, K, 1, 0, T, dst, stream);
    }
    const int rows_max = (T + G - 1) / G;
    const size_t need = (size_t)G * rows_max * N * 2;
    if (!comm->open || comm->win_bytes < need)
        return fail(HG_E_INVALID, "out-proj reduce-scatter needs an open peer window of %zu bytes", need);
    unsigned long long *fl[kMaxOuts];
    for (int k = 0; k < G; ++k) fl[k] = (unsigned long long *)comm->peer[k];
    unsigned long long *mine = (unsigned long long *)comm->win;
    // entry: no rank overwrites a receive slot its owner may still be reducing
    hg_status s = launch_peer_barrier(fl, mine, comm->rank, G, ++comm->epoch, stream);
    if (s) return s;
    uint16_t *dst[kMaxOuts];
    for (int k = 0; k < G; ++k) dst[k] = (uint16_t *)(comm->peer[k] + kWinHdr);
    s = launch_out_proj((const uint16_t *)o_local, (const uint16_t *)w_local, T, N, K, G, comm->rank, rows_max, dst,
                        stream);
    if (s) return s;
    s = launch_peer_barrier(fl, mine, comm->rank, G, ++comm->epoch, stream);   // every partial row has landed
    if (s) return s;
    const int r0 = (comm->rank * T) / G, r1 = ((comm->rank + 1) * T) / G;
    return launch_rs_reduce((const uint16_t *)(comm->win + kWinHdr), (uint16_t *)y_shard, r1 - r0, rows_max, N, G,
                            stream);
}

extern "C" hg_status hg_hybrid_attention_tp_proj_workspace_size(const hg_kv_pool *pool, const hg_comm *comm,
                                                                const hg_batch *batch, int32_t H_q, size_t *bytes) {
    if (!pool || !comm || !batch || !bytes) return fail(HG_E_INVALID, "NULL argument");
    if (H_q % comm->world) return fail(HG_E_INVALID, "num_q_heads %d not divisible by world %d", H_q, comm->world);
    size_t attn = 0;
    hg_status s = hg_hybrid_attention_workspace_size(pool, batch, H_q / comm->world, &attn);
    if (s) return s;
    int64_t T = 0;
    for (int i = 0; i < batch->num_reqs; ++i) T += batch->new_len[i];
    *bytes = al256(attn) + al256((size_t)T * (H_q / comm->world) * pool_head_dim(pool) * 2);
    return HG_OK;
}

extern "C" hg_status hg_hybrid_attention_tp_proj(hg_kv_pool *pool, hg_comm *comm, const hg_batch *batch, int32_t H_q,
                                                 const void *q_local, const void *w_local, int32_t N, void *y_shard,
                                                 void *workspace, size_t workspace_bytes, void *stream) {
    if (!pool || !comm || !batch) return fail(HG_E_INVALID, "NULL argument");
    size_t need = 0;
    hg_status s = hg_hybrid_attention_tp_proj_workspace_size(pool, comm, batch, H_q, &need);
    if (s) return s;
    if (!workspace || workspace_bytes < need)
        return fail(HG_E_INVALID, "workspace too small (%zu < %zu)", workspace_bytes, need);
    const int Hl = H_q / comm->world, d = pool_head_dim(pool);
    int64_t T = 0;
    for (int i = 0; i < batch->num_reqs; ++i) T += batch->new_len[i];
    size_t attn = 0;
    s = hg_hybrid_attention_workspace_size(pool, batch, Hl, &attn);
    if (s) return s;
    uint16_t *o_local = (uint16_t *)((uint8_t *)workspace + al256(attn));   // [T][Hl][d]
    s = hg_hybrid_attention(pool, batch, Hl, q_local, o_local, nullptr, workspace, attn, stream);
    if (s) return s;
    return hg_out_proj_rs(comm, (int32_t)T, Hl * d, N, o_local, w_local, y_shard, stream);
}
