// api.cpp -- C ABI entry points: KV pool + allocator, append, hybrid attention
// orchestration (plan -> pinned staging -> H2D -> kernels), e2e host step,
// batch indices, predictor (Eq. 1 / Eq. 2 linear regression).
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <set>
#include <vector>

#include "hg_internal.h"

using namespace hg;

namespace hg {
bool make_tensor_maps(hg_kv_pool *pool);  // tc_attn.cu
}

struct hg_kv_pool {
    hg_kv_pool_desc desc{};
    std::vector<int32_t> ref;
    std::set<int32_t> free_ids;
    int num_sms = 148;
    // pinned staging ring for per-call descriptors
    struct Stage {
        void *host = nullptr;
        size_t cap = 0;
        cudaEvent_t ev = nullptr;
        bool pending = false;
    };
    static constexpr int kRing = 8;  // descriptor copies in flight: the host may plan ~4 calls ahead
    Stage ring[kRing];
    int ring_pos = 0;
    alignas(64) unsigned char tmap_k[128];
    alignas(64) unsigned char tmap_v[128];
    bool tmap_ok = false;
    hg_plan_stats last{};
    Plan plan;  // reused storage
    // host step planned ahead (hg_hybrid_step_host_plan): the plan, for which batch
    Plan plan_ahead;
    bool ahead_ok = false;
    const hg_batch *ahead_batch = nullptr;
    int32_t ahead_Hq = 0;
    uint64_t ahead_fp = 0;
    // side stream: the split-K kernel runs beside the tcgen05 kernel (fork/join by events)
    cudaStream_t side = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    // hg_hybrid_step_host: copy stream for the two input waves, their events, and
    // the prefill wave's tcgen05 stream (highest priority) with its done events
    cudaStream_t h2d = nullptr, side_hi = nullptr;
    cudaEvent_t ev_in0 = nullptr, ev_in1 = nullptr, ev_tc = nullptr, ev_d2h = nullptr;
    // fused step: the append runs on `side` while the descriptors upload
    cudaEvent_t ev_pre = nullptr, ev_app = nullptr;
    // Device descriptor slots (library-owned): a call's descriptor image goes up on
    // the copy stream `cp`, which waits only for the kernels of the call that last
    // used the slot -- not for the caller's queued work -- so the upload of step
    // k+1 overlaps step k's kernels (the host plans ahead of the GPU).
    struct DSlot {
        void *dev = nullptr;
        size_t cap = 0;
        cudaEvent_t ready = nullptr, done = nullptr;
        bool used = false;
    };
    static constexpr int kDRing = 4;
    DSlot dring[kDRing];
    int dpos = 0;
    cudaStream_t cp = nullptr;
    // fused append inside the tcgen05 kernel: device counter of finished shares and
    // the host's running total of the shares launched (each call waits for its own)
    unsigned long long *app_cnt = nullptr;
    unsigned long long app_total = 0;
    // ... and per request (background append): device counts and the host's targets
    unsigned long long *app_req_cnt = nullptr;
    std::vector<unsigned long long> app_req_total;
};

namespace hg {
void *pool_tmap_k(hg_kv_pool *p) { return p->tmap_k; }
void *pool_tmap_v(hg_kv_pool *p) { return p->tmap_v; }
const hg_kv_pool_desc &pool_desc(hg_kv_pool *p) { return p->desc; }
void pool_set_tmap_ok(hg_kv_pool *p, bool ok) { p->tmap_ok = ok; }
}  // namespace hg

static hg_status cuda_check(cudaError_t e, const char *what) {
    if (e == cudaSuccess) return HG_OK;
    return fail(HG_E_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

// Surface errors from earlier asynchronous launches (header contract).
static hg_status sticky_check() {
    cudaError_t e = cudaPeekAtLastError();
    if (e != cudaSuccess) {
        cudaGetLastError();
        return fail(HG_E_CUDA, "earlier CUDA error: %s", cudaGetErrorString(e));
    }
    return HG_OK;
}

// Copy `bytes` of host data to `dst` on `stream` through a pinned staging buffer.
// Copy `bytes` to device memory `dst` on `st` through the next pinned staging slot;
// `fill` writes the bytes into the slot (so an image can be assembled in place).
template <typename Fill>
static hg_status stage_h2d_fill(hg_kv_pool *pool, void *dst, size_t bytes, cudaStream_t st, const Fill &fill) {
    if (bytes == 0) return HG_OK;
    auto &s = pool->ring[pool->ring_pos];
    pool->ring_pos = (pool->ring_pos + 1) % hg_kv_pool::kRing;
    if (s.pending) {
        hg_status r = cuda_check(cudaEventSynchronize(s.ev), "staging event sync");
        if (r) return r;
        s.pending = false;
    }
    if (s.cap < bytes) {
        if (s.host) cudaFreeHost(s.host);
        size_t cap = std::max<size_t>(bytes * 2, 1 << 16);
        hg_status r = cuda_check(cudaHostAlloc(&s.host, cap, cudaHostAllocDefault), "cudaHostAlloc");
        if (r) { s.host = nullptr; s.cap = 0; return r; }
        s.cap = cap;
    }
    if (!s.ev) {
        hg_status r = cuda_check(cudaEventCreateWithFlags(&s.ev, cudaEventDisableTiming), "event create");
        if (r) return r;
    }
    fill((uint8_t *)s.host);
    hg_status r = cuda_check(cudaMemcpyAsync(dst, s.host, bytes, cudaMemcpyHostToDevice, st), "H2D descriptors");
    if (r) return r;
    r = cuda_check(cudaEventRecord(s.ev, st), "event record");
    if (r) return r;
    s.pending = true;
    return HG_OK;
}

static hg_status stage_h2d(hg_kv_pool *pool, void *dst, const void *src, size_t bytes, cudaStream_t st) {
    return stage_h2d_fill(pool, dst, bytes, st, [&](uint8_t *h) { memcpy(h, src, bytes); });
}

// Upload a call's descriptor image into the next device slot on the copy stream
// and make `st` wait for it.  The copy waits (on the GPU) only for the kernels
// of the call that used the slot before; the caller records `done` after its
// last kernel (DescDone).
template <typename Fill>
// `cp`: the copy stream (NULL: the pool's own).  The host step passes its input copy
// stream, so the descriptors go up in order with the input waves: on a separate stream
// the copy engine may run a later wave's megabytes first and hold the kernels back.
static hg_status stage_desc(hg_kv_pool *pool, const Fill &fill, size_t bytes, cudaStream_t st, void **dev,
                            hg_kv_pool::DSlot **slot, cudaStream_t cp = nullptr) {
    hg_status s = HG_OK;
    if (!pool->cp) s = cuda_check(cudaStreamCreateWithFlags(&pool->cp, cudaStreamNonBlocking), "copy stream");
    if (s) return s;
    if (!cp) cp = pool->cp;
    hg_kv_pool::DSlot &d = pool->dring[pool->dpos];
    pool->dpos = (pool->dpos + 1) % hg_kv_pool::kDRing;
    for (cudaEvent_t *e : {&d.ready, &d.done})
        if (!*e && !s) s = cuda_check(cudaEventCreateWithFlags(e, cudaEventDisableTiming), "event create");
    if (s) return s;
    if (d.cap < bytes) {
        if (d.dev) {
            if (d.used) cudaEventSynchronize(d.done);
            cudaFree(d.dev);
            d.dev = nullptr;
            d.cap = 0;
            d.used = false;
        }
        const size_t cap = std::max<size_t>(bytes * 3 / 2, 1 << 16);
        s = cuda_check(cudaMalloc(&d.dev, cap), "cudaMalloc(descriptors)");
        if (s) { d.dev = nullptr; return s; }
        d.cap = cap;
    }
    if (d.used) s = cuda_check(cudaStreamWaitEvent(cp, d.done, 0), "descriptor slot wait");
    if (!s) s = stage_h2d_fill(pool, d.dev, bytes, cp, fill);   // the image is assembled in the pinned slot
    if (!s) s = cuda_check(cudaEventRecord(d.ready, cp), "descriptor ready record");
    if (!s) s = cuda_check(cudaStreamWaitEvent(st, d.ready, 0), "descriptor ready wait");
    if (s) return s;
    *dev = d.dev;
    *slot = &d;
    return HG_OK;
}

// Records the slot's `done` on the caller's stream when the call's launches are
// over (every kernel that reads the descriptors is ordered before it on `st`).
struct DescDone {
    hg_kv_pool::DSlot *slot = nullptr;
    cudaStream_t st = nullptr;
    ~DescDone() {
        if (slot && cudaEventRecord(slot->done, st) == cudaSuccess) slot->used = true;
    }
};

// ---------------------------------------------------------------------------
// pool + allocator
// ---------------------------------------------------------------------------
extern "C" hg_status hg_kv_pool_create(const hg_kv_pool_desc *d, hg_kv_pool **out) {
    if (!d || !out) return fail(HG_E_INVALID, "NULL argument");
    if (d->num_blocks < 1 || d->num_kv_heads < 1) return fail(HG_E_INVALID, "num_blocks and num_kv_heads must be >= 1");
    if (d->block_size != kBlock) return fail(HG_E_UNSUPPORTED, "block_size %d (this build: %d)", d->block_size, kBlock);
    if (d->head_dim != 64 && d->head_dim != 128) return fail(HG_E_UNSUPPORTED, "head_dim %d (64 or 128)", d->head_dim);
    if (!d->k_cache || !d->v_cache || ((uintptr_t)d->k_cache & 15) || ((uintptr_t)d->v_cache & 15))
        return fail(HG_E_INVALID, "k_cache / v_cache must be non-NULL and 16-byte aligned");
    hg_kv_pool *p = new hg_kv_pool();
    p->desc = *d;
    p->ref.assign((size_t)d->num_blocks, 0);
    for (int32_t i = 0; i < d->num_blocks; ++i) p->free_ids.insert(p->free_ids.end(), i);
    int sms = 0;
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, d->device) == cudaSuccess && sms > 0)
        p->num_sms = sms;
    else
        cudaGetLastError();
    p->tmap_ok = make_tensor_maps(p);
    *out = p;
    return HG_OK;
}

extern "C" hg_status hg_kv_pool_destroy(hg_kv_pool *p) {
    if (!p) return HG_OK;
    for (auto &s : p->ring) {
        if (s.pending) cudaEventSynchronize(s.ev);
        if (s.host) cudaFreeHost(s.host);
        if (s.ev) cudaEventDestroy(s.ev);
    }
    if (p->side) {
        cudaStreamSynchronize(p->side);
        cudaStreamDestroy(p->side);
    }
    if (p->ev_fork) cudaEventDestroy(p->ev_fork);
    if (p->ev_join) cudaEventDestroy(p->ev_join);
    for (cudaStream_t s : {p->h2d, p->side_hi})
        if (s) {
            cudaStreamSynchronize(s);
            cudaStreamDestroy(s);
        }
    for (cudaEvent_t e : {p->ev_in0, p->ev_in1, p->ev_tc, p->ev_d2h, p->ev_pre, p->ev_app})
        if (e) cudaEventDestroy(e);
    for (auto &d : p->dring) {
        if (d.used) cudaEventSynchronize(d.done);
        if (d.dev) cudaFree(d.dev);
        for (cudaEvent_t e : {d.ready, d.done})
            if (e) cudaEventDestroy(e);
    }
    if (p->cp) {
        cudaStreamSynchronize(p->cp);
        cudaStreamDestroy(p->cp);
    }
    if (p->app_cnt) cudaFree(p->app_cnt);
    if (p->app_req_cnt) cudaFree(p->app_req_cnt);
    delete p;
    return HG_OK;
}

extern "C" hg_status hg_kv_alloc(hg_kv_pool *p, int32_t n, int32_t *out_ids) {
    if (!p || (n > 0 && !out_ids) || n < 0) return fail(HG_E_INVALID, "bad arguments");
    if ((size_t)n > p->free_ids.size())
        return fail(HG_E_OOM, "need %d blocks, free %zu", n, p->free_ids.size());
    auto it = p->free_ids.begin();
    for (int32_t k = 0; k < n; ++k) {
        out_ids[k] = *it;
        p->ref[*it] = 1;
        it = p->free_ids.erase(it);
    }
    return HG_OK;
}

extern "C" hg_status hg_kv_retain(hg_kv_pool *p, const int32_t *ids, int32_t n) {
    if (!p || n < 0 || (n > 0 && !ids)) return fail(HG_E_INVALID, "bad arguments");
    for (int32_t k = 0; k < n; ++k)
        if (ids[k] < 0 || ids[k] >= p->desc.num_blocks || p->ref[ids[k]] == 0)
            return fail(HG_E_INVALID, "retain of unallocated block %d", ids[k]);
    for (int32_t k = 0; k < n; ++k) p->ref[ids[k]]++;
    return HG_OK;
}

extern "C" hg_status hg_kv_release(hg_kv_pool *p, const int32_t *ids, int32_t n) {
    if (!p || n < 0 || (n > 0 && !ids)) return fail(HG_E_INVALID, "bad arguments");
    std::vector<std::pair<int32_t, int32_t>> need;
    for (int32_t k = 0; k < n; ++k) {
        if (ids[k] < 0 || ids[k] >= p->desc.num_blocks) return fail(HG_E_INVALID, "release of block %d out of range", ids[k]);
        need.push_back({ids[k], 1});
    }
    std::sort(need.begin(), need.end());
    for (size_t a = 0; a < need.size();) {
        size_t b = a;
        int cnt = 0;
        while (b < need.size() && need[b].first == need[a].first) cnt += need[b++].second;
        if (p->ref[need[a].first] < cnt) return fail(HG_E_INVALID, "release of block %d below refcount 0", need[a].first);
        a = b;
    }
    for (int32_t k = 0; k < n; ++k)
        if (--p->ref[ids[k]] == 0) p->free_ids.insert(ids[k]);
    return HG_OK;
}

extern "C" int32_t hg_kv_num_free(const hg_kv_pool *p) { return p ? (int32_t)p->free_ids.size() : 0; }

extern "C" int32_t hg_kv_refcount(const hg_kv_pool *p, int32_t id) {
    if (!p || id < 0 || id >= p->desc.num_blocks) return -1;
    return p->ref[id];
}

// ---------------------------------------------------------------------------
// a.1 indices
// ---------------------------------------------------------------------------
extern "C" hg_status hg_batch_indices(const hg_kv_pool *pool, const hg_batch *batch, int32_t *cu_q,
                                      int32_t *kv_len, int64_t *slot, int32_t *prefix_group) {
    if (!pool) return fail(HG_E_INVALID, "pool is NULL");
    BatchView v;
    hg_status s = view_batch(batch, &v);
    if (s) return s;
    s = validate(v, pool->desc.block_size, pool->desc.num_blocks, -1, 0, false);
    if (s) return s;
    const int B = pool->desc.block_size;
    int64_t t = 0;
    if (cu_q) cu_q[0] = 0;
    for (int i = 0; i < v.R; ++i) {
        if (cu_q) cu_q[i + 1] = cu_q[i] + v.n[i];
        if (kv_len) kv_len[i] = v.c[i] + v.n[i];
        for (int j = 0; j < v.n[i]; ++j, ++t) {
            int64_t pos = (int64_t)v.c[i] + j;
            if (slot) slot[t] = (int64_t)v.bt[(int64_t)i * v.W + pos / B] * B + pos % B;
        }
    }
    if (prefix_group) {
        std::vector<int32_t> g;
        prefix_groups(v, &g);
        memcpy(prefix_group, g.data(), sizeof(int32_t) * (size_t)v.R);
    }
    return HG_OK;
}

// ---------------------------------------------------------------------------
// a.3 append
// ---------------------------------------------------------------------------
// Small device scratch for append slots when they do not fit the kernel
// parameters (pool-independent, grows on demand).  Appends may come on different
// streams: each staging copy waits (stream-ordered) for the previous append
// kernel that read the buffer, whatever its stream.
static thread_local void *g_slot_dev = nullptr;
static thread_local size_t g_slot_cap = 0;
static thread_local cudaEvent_t g_slot_ev = nullptr;   // recorded after the last kernel that read g_slot_dev

static hg_status slot_buffer(size_t need, cudaStream_t st) {
    hg_status s = HG_OK;
    if (!g_slot_ev) s = cuda_check(cudaEventCreateWithFlags(&g_slot_ev, cudaEventDisableTiming), "slot event");
    if (s) return s;
    if (g_slot_cap < need) {
        if (g_slot_dev) {
            cudaEventSynchronize(g_slot_ev);
            cudaFree(g_slot_dev);
            g_slot_dev = nullptr;
            g_slot_cap = 0;
        }
        const size_t cap = std::max<size_t>(need * 2, 1 << 16);
        s = cuda_check(cudaMalloc(&g_slot_dev, cap), "cudaMalloc(slots)");
        if (s) { g_slot_dev = nullptr; return s; }
        g_slot_cap = cap;
    }
    return cuda_check(cudaStreamWaitEvent(st, g_slot_ev, 0), "slot buffer wait");
}

static hg_status append_impl(hg_kv_pool *pool, const BatchView &v, const void *k_new, const void *v_new,
                             cudaStream_t st) {
    const int B = pool->desc.block_size;
    int64_t T = 0;
    for (int i = 0; i < v.R; ++i) T += v.n[i];
    if (T == 0) return HG_OK;
    static thread_local std::vector<int64_t> slot;
    slot.resize((size_t)T);
    int64_t t = 0;
    for (int i = 0; i < v.R; ++i)
        for (int j = 0; j < v.n[i]; ++j, ++t) {
            int64_t pos = (int64_t)v.c[i] + j;
            slot[t] = (int64_t)v.bt[(int64_t)i * v.W + pos / B] * B + pos % B;
        }
    auto *kc = (uint16_t *)pool->desc.k_cache, *vc = (uint16_t *)pool->desc.v_cache;
    if (T <= kParamSlots)   // slots in the kernel parameters: no staging buffer, no H2D
        return launch_append_param((const uint16_t *)k_new, (const uint16_t *)v_new, kc, vc, slot.data(), (int)T,
                                   pool->desc.num_kv_heads, pool->desc.head_dim, st);
    hg_status s = slot_buffer(sizeof(int64_t) * (size_t)T, st);
    if (!s) s = stage_h2d(pool, g_slot_dev, slot.data(), sizeof(int64_t) * (size_t)T, st);
    if (!s) s = launch_append((const uint16_t *)k_new, (const uint16_t *)v_new, kc, vc, (const int64_t *)g_slot_dev,
                              (int)T, pool->desc.num_kv_heads, pool->desc.head_dim, st);
    if (!s) s = cuda_check(cudaEventRecord(g_slot_ev, st), "slot event record");
    return s;
}

static hg_status rope_args(const hg_rope *r, int d, RopeArgs *out) {
    const int rot = r->rotary_dim ? r->rotary_dim : d;
    if (!(r->theta > 0) || rot <= 0 || rot > d || rot % 16 || rot > 256)
        return fail(HG_E_INVALID, "rope: theta %g, rotary_dim %d (head_dim %d): need theta > 0, R %% 16 == 0, R <= d",
                    r->theta, r->rotary_dim, d);
    out->theta = r->theta;
    out->rot = rot;
    return HG_OK;
}

extern "C" hg_status hg_kv_append(hg_kv_pool *pool, const hg_batch *batch, const void *k_new,
                                  const void *v_new, void *stream) {
    if (!pool) return fail(HG_E_INVALID, "pool is NULL");
    BatchView v;
    hg_status s = view_batch(batch, &v);
    if (s) return s;
    s = validate(v, pool->desc.block_size, pool->desc.num_blocks, -1, 0, true);
    if (s) return s;
    s = sticky_check();
    if (s) return s;
    int64_t T = 0;
    for (int i = 0; i < v.R; ++i) T += v.n[i];
    if (T == 0) return HG_OK;
    if (!k_new || !v_new) return fail(HG_E_INVALID, "k_new / v_new NULL");
    return append_impl(pool, v, k_new, v_new, (cudaStream_t)stream);
}

extern "C" hg_status hg_kv_append_rope(hg_kv_pool *pool, const hg_batch *batch, const void *k_new,
                                       const void *v_new, const hg_rope *rope, void *stream) {
    if (!pool || !rope) return fail(HG_E_INVALID, "pool / rope is NULL");
    RopeArgs ra;
    hg_status s = rope_args(rope, pool->desc.head_dim, &ra);
    if (s) return s;
    BatchView v;
    s = view_batch(batch, &v);
    if (s) return s;
    s = validate(v, pool->desc.block_size, pool->desc.num_blocks, -1, 0, true);
    if (s) return s;
    s = sticky_check();
    if (s) return s;
    int64_t T = 0;
    for (int i = 0; i < v.R; ++i) T += v.n[i];
    if (T == 0) return HG_OK;
    if (!k_new || !v_new) return fail(HG_E_INVALID, "k_new / v_new NULL");
    const int B = pool->desc.block_size;
    // staged: slot int64 [T], then position int32 [T]
    std::vector<uint8_t> img((size_t)T * 12);
    int64_t *slot = (int64_t *)img.data();
    int32_t *pos = (int32_t *)(img.data() + (size_t)T * 8);
    int64_t t = 0;
    for (int i = 0; i < v.R; ++i)
        for (int j = 0; j < v.n[i]; ++j, ++t) {
            const int64_t p = (int64_t)v.c[i] + j;
            slot[t] = (int64_t)v.bt[(int64_t)i * v.W + p / B] * B + p % B;
            pos[t] = (int32_t)p;
        }
    cudaStream_t st = (cudaStream_t)stream;
    s = slot_buffer(img.size(), st);
    if (!s) s = stage_h2d(pool, g_slot_dev, img.data(), img.size(), st);
    if (!s) s = launch_rope_append((const uint16_t *)k_new, (const uint16_t *)v_new, (uint16_t *)pool->desc.k_cache,
                                   (uint16_t *)pool->desc.v_cache, (const int64_t *)g_slot_dev,
                                   (const int32_t *)((uint8_t *)g_slot_dev + (size_t)T * 8), (int)T,
                                   pool->desc.num_kv_heads, pool->desc.head_dim, ra, st);
    if (!s) s = cuda_check(cudaEventRecord(g_slot_ev, st), "slot event record");
    return s;
}

// ---------------------------------------------------------------------------
// a.1-a.7 hybrid attention
// ---------------------------------------------------------------------------
static hg_status ensure_side(hg_kv_pool *pool) {
    if (pool->side) return HG_OK;
    hg_status s = cuda_check(cudaStreamCreateWithFlags(&pool->side, cudaStreamNonBlocking), "side stream");
    if (s) return s;
    s = cuda_check(cudaEventCreateWithFlags(&pool->ev_fork, cudaEventDisableTiming), "fork event");
    if (s) return s;
    return cuda_check(cudaEventCreateWithFlags(&pool->ev_join, cudaEventDisableTiming), "join event");
}

// High-priority stream for the tcgen05 tiles when they run beside split-K
// (their CTAs need whole SMs: at equal priority split-K's queued CTAs can take
// every SM that frees up), and the event that joins it.
static hg_status ensure_hi(hg_kv_pool *pool) {
    if (pool->side_hi) return HG_OK;
    int lo = 0, hi = 0;
    hg_status s = cuda_check(cudaDeviceGetStreamPriorityRange(&lo, &hi), "priority range");
    if (!s) s = cuda_check(cudaStreamCreateWithPriority(&pool->side_hi, cudaStreamNonBlocking, hi), "tc stream");
    if (!s) s = cuda_check(cudaEventCreateWithFlags(&pool->ev_tc, cudaEventDisableTiming), "tc event");
    return s;
}

// Pipelined host step (hg_hybrid_step_host): the inputs arrive in two waves on
// a copy stream -- wave 0 = the decode rows' Q/K/V, wave 1 = the prefill-chunk
// rows' -- and each wave's append and attention start as soon as it lands.
struct StepPipe {
    cudaEvent_t in0 = nullptr, in1 = nullptr;   // recorded on the copy stream after each wave
    cudaStream_t side = nullptr;                // stream of the wave-1 work (append + tcgen05)
    cudaEvent_t tc_done = nullptr;              // recorded on `side` after the tcgen05 kernel
    std::function<hg_status(int)> enqueue_wave; // issues wave w's copies and records in0 / in1: wave 0 right
                                                // after the descriptor upload (which must not queue behind
                                                // the inputs on the copy engine), wave 1 after the split-K
                                                // launch (so that launch is not delayed by the host)
    bool planned = false;                       // pool->plan already holds this batch's validated plan
    bool used = false;                          // out: the call was split into waves
    cudaStream_t copy = nullptr;                // stream of the input copies (the descriptors follow them)
    uint16_t *zc_out = nullptr;                 // device-visible pinned host O: split-K and the combine
                                                // store their final rows there (zero-copy result)
};
static PlanOpts plan_opts(const hg_kv_pool *pool, const hg_attn_opts *o) {
    PlanOpts po;
    po.num_sms = pool->num_sms;
    if (o) {
        po.split_tokens = o->split_tokens;
        po.prefix_pass = !o->disable_prefix_pass;
        po.use_tc = !o->disable_tc;
        po.split_prefill = !o->disable_prefill_split;
        po.route = o->route;
        if (o->num_sms > 0) po.num_sms = o->num_sms;
    }
    return po;
}

static hg_status plan_call(hg_kv_pool *pool, const hg_batch *batch, int32_t H_q, const hg_attn_opts *o,
                           BatchView *v, Plan *plan, bool append = false) {
    hg_status s = view_batch(batch, v);
    if (s) return s;
    s = validate(*v, pool->desc.block_size, pool->desc.num_blocks, H_q, pool->desc.num_kv_heads, append);
    if (s) return s;
    PlanOpts po = plan_opts(pool, o);
    if (!pool->tmap_ok) po.use_tc = false;
    return build_plan(*v, H_q, pool->desc.num_kv_heads, pool->desc.head_dim, po, plan);
}

extern "C" hg_status hg_hybrid_attention_workspace_size(const hg_kv_pool *pool, const hg_batch *batch,
                                                        int32_t num_q_heads, size_t *bytes) {
    if (!pool || !bytes) return fail(HG_E_INVALID, "NULL argument");
    BatchView v;
    Plan plan;
    hg_status s = plan_call(const_cast<hg_kv_pool *>(pool), batch, num_q_heads, nullptr, &v, &plan);
    if (s) return s;
    *bytes = plan.total_bytes;
    return HG_OK;
}

// k_new / v_new non-NULL: fused step, the append kernel runs first from the same
// descriptors (slots computed on the device).
// outs non-NULL: O goes to every destination it lists (peer-window all-gather)
// instead of `out`.
static hg_status attention_impl(hg_kv_pool *pool, const hg_batch *batch, int32_t H_q, const void *q, void *out,
                                float *lse, void *ws, size_t ws_bytes, cudaStream_t st, const hg_attn_opts *o,
                                bool fused = false, const void *k_new = nullptr, const void *v_new = nullptr,
                                const OutSpec *outs = nullptr, StepPipe *pipe = nullptr, bool planned = false) {
    BatchView v;
    Plan &plan = pool->plan;
    hg_status s = (planned || (pipe && pipe->planned)) ? view_batch(batch, &v)
                                                       : plan_call(pool, batch, H_q, o, &v, &plan, fused);
    if (s) return s;
    s = sticky_check();
    if (s) return s;
    if (plan.T == 0) {
        pool->last = hg_plan_stats{};
        return HG_OK;
    }
    if (!q || (!out && !outs)) return fail(HG_E_INVALID, "q / out NULL");
    RopeArgs ra;
    if (o && o->rope) {
        if (!fused) return fail(HG_E_INVALID, "rope is applied in the hg_hybrid_step prologue only");
        s = rope_args(o->rope, pool->desc.head_dim, &ra);
        if (s) return s;
    }
    if (fused && (!k_new || !v_new)) return fail(HG_E_INVALID, "k_new / v_new NULL");
    if (!ws || ws_bytes < plan.total_bytes)
        return fail(HG_E_INVALID, "workspace %zu bytes < required %zu", ws_bytes, plan.total_bytes);
    // Two waves -- decode rows (append + split-K on the caller's stream) and
    // prefill-chunk rows (append + tcgen05 on the high-priority stream) -- when
    // wave 0's work reads no wave-1 input: every prefill chunk is on the tcgen05
    // tiles (the prefix-group tiles read only cached keys and decode-row Q).
    // Split-K then waits only for the decode rows' append; the host step
    // (pipe != NULL) also feeds each wave from its own H2D copies.
    StepPipe local;
    {
        static const bool serial = getenv("HG_E2E_SERIAL") != nullptr;   // A/B switches: one wave
        // device-buffer step: off by default -- measured slower on c1 (0.460 vs 0.4555 ms:
        // the decode rows' append alone still takes ~5 us, and the tiles, started
        // later, then overlap more of split-K); HG_STEP_WAVES=1 turns it on
        static const bool no_waves = getenv("HG_STEP_WAVES") == nullptr;
        bool ok = fused && !ra.rot && plan.n_tc_prefill() > 0 && !plan.sk.empty();
        for (size_t k = 0; ok && k < plan.sk.size(); ++k) ok = v.n[plan.sk[k].req] == 1;
        if (pipe) {
            pipe->used = ok && !serial;
        } else if (ok && !no_waves) {
            s = ensure_hi(pool);
            if (s) return s;
            local.side = pool->side_hi;
            local.tc_done = pool->ev_tc;
            local.used = true;
            pipe = &local;
        }
        if (pipe && pipe->used)
            for (TokDev &tk : plan.tok) tk.wave = v.n[tk.req] > 1 ? 1 : 0;
        // zero-copy result only where every row is written either by split-K / the
        // combine (to the host) or by the tcgen05 kernel of the two-wave step (its rows
        // are copied back on their own): not when one launch mixes both into one copy
        if (pipe && pipe->zc_out && !pipe->used && !plan.tc.empty()) pipe->zc_out = nullptr;
    }
    // tcgen05 route: the append runs inside the tcgen05 kernel, each CTA writing
    // its share of the new tokens (<= ~256 KB of K+V per CTA), and a TMA producer
    // waits only before the first tile holding new keys -- no append kernel and no
    // launch in front of the tiles.  Not with the rope prologue or a peer-window
    // entry barrier (those ride in the append kernel).
    static const bool no_tc_append = getenv("HG_NO_TC_APPEND") != nullptr;   // A/B switch
    static const bool no_bg_append = getenv("HG_NO_BG_APPEND") != nullptr;   // A/B switch
    const int64_t tc_grid = std::max<int64_t>(1, std::min<int64_t>((int64_t)plan.tc.size(), plan.tc_ctas));
    const bool tc_append = fused && !ra.rot && !pipe && !plan.tc.empty() && !(outs && outs->bar_world > 0) &&
                           !no_tc_append &&
                           (int64_t)plan.T * pool->desc.num_kv_heads * pool->desc.head_dim * 4 <= tc_grid * (256 << 10);
    // Where: in the prologue (all 384 threads, ~HBM rate, every pipeline waits for
    // it) or in the background on each CTA's idle warp, request by request in the
    // order the tiles need them (each request's tokens sliced over the grid, ~5 KB/us
    // per CTA), a TMA producer waiting only for its own item's request.  Each CTA's
    // items are reordered so the one with the most cached-prefix tiles before its first
    // new key comes first (the CTA's load is unchanged); a request's need time is the
    // earliest (item start + cached-prefix tiles) over the items reading its new keys.
    // Background when every request is appended, at the grid's aggregate rate, before
    // its need time.
    bool app_bg = false;
    int32_t app_head = -1;
    if (tc_append && !no_bg_append && (int64_t)plan.tc_off.size() == tc_grid + 1) {
        constexpr double kTileUs = 1.5, kItemUs = 2.0, kBgBytesPerUs = 5.0e3, kSlackUs = 5.0;
        auto lead_tiles = [](const TcItem &it) {
            const int64_t nkt = (it.k1 - it.k0 + kTcKeys - 1) / kTcKeys;
            const int64_t before = it.cnew <= it.k0 ? 0 : (int64_t)(it.cnew - it.k0) / kTcKeys;
            return std::min(nkt, before);
        };
        static thread_local std::vector<double> need;
        need.assign((size_t)v.R, 1e30);   // decode rows: split-K reads their new keys from the inputs
        for (int64_t b = 0; b < tc_grid; ++b) {
            TcItem *a = plan.tc.data() + plan.tc_off[b], *e = plan.tc.data() + plan.tc_off[b + 1];
            std::stable_sort(a, e, [&](const TcItem &x, const TcItem &y) { return lead_tiles(x) > lead_tiles(y); });
            double at = 0;
            for (TcItem *it = a; it < e; ++it) {
                const int64_t nkt = (it->k1 - it->k0 + kTcKeys - 1) / kTcKeys;
                if (it->mode == 0 && it->cnew < it->k1) {
                    const int r = plan.tok[it->t0].req;
                    need[r] = std::min(need[r], at + (double)lead_tiles(*it) * kTileUs);
                }
                at += (double)nkt * kTileUs + kItemUs;
            }
        }
        static thread_local std::vector<int32_t> order;
        order.resize((size_t)v.R);
        for (int i = 0; i < v.R; ++i) order[i] = i;
        std::stable_sort(order.begin(), order.end(), [&](int32_t x, int32_t y) { return need[x] < need[y]; });
        const double bytes_per_tok = 4.0 * pool->desc.num_kv_heads * pool->desc.head_dim;   // K + V
        double done_us = 0;
        app_bg = true;
        for (int32_t r : order) {
            done_us += (double)v.n[r] * bytes_per_tok / (kBgBytesPerUs * (double)tc_grid);
            if (need[r] < 1e29 && done_us + kSlackUs > need[r]) {
                app_bg = false;
                break;
            }
        }
        if (app_bg) {
            if ((int64_t)pool->app_req_total.size() < v.R) {   // grow the per-request counters
                if (pool->app_req_cnt) cudaFree(pool->app_req_cnt);
                pool->app_req_cnt = nullptr;
                const size_t cap = std::max<size_t>(256, (size_t)v.R * 2);
                s = cuda_check(cudaMalloc(&pool->app_req_cnt, cap * 8), "cudaMalloc(request counters)");
                if (!s) s = cuda_check(cudaMemset(pool->app_req_cnt, 0, cap * 8), "memset(request counters)");
                if (!s) s = cuda_check(cudaDeviceSynchronize(), "request counters init");
                if (s) { if (pool->app_req_cnt) cudaFree(pool->app_req_cnt); pool->app_req_cnt = nullptr;
                         pool->app_req_total.clear(); return s; }
                pool->app_req_total.assign(cap, 0ull);
            }
            for (int k = 0; k < v.R; ++k) {
                const int32_t r = order[k];
                plan.reqs[r].app_next = k + 1 < v.R ? order[k + 1] : -1;
                pool->app_req_total[r] += (unsigned long long)tc_grid;   // one count per CTA
                plan.reqs[r].app_tgt = pool->app_req_total[r];
            }
            app_head = v.R > 0 ? order[0] : -1;
        }
    }
    // one image of all descriptors -> one pinned H2D copy, assembled in the staging slot
    // (alignment gaps are never read; the in-kernel counters at off_cnt.. are zeroed)
    auto build_img = [&](uint8_t *img) {
        auto put = [&](size_t off, const void *src, size_t n) { if (n) memcpy(img + off, src, n); };
        put(plan.off_reqs, plan.reqs.data(), sizeof(ReqDev) * plan.reqs.size());
        for (int i = 0; i < v.R; ++i)   // block tables: straight from the caller's rows
            put(plan.off_bt + sizeof(int32_t) * (size_t)plan.reqs[i].bt_off, v.bt + (int64_t)i * v.W,
                sizeof(int32_t) * (size_t)((v.c[i] + v.n[i] + pool->desc.block_size - 1) / pool->desc.block_size));
        put(plan.off_sk, plan.sk.data(), sizeof(SkItem) * plan.sk.size());
        put(plan.off_tc, plan.tc.data(), sizeof(TcItem) * plan.tc.size());
        put(plan.off_rows, plan.tc_tok.data(), sizeof(int32_t) * plan.tc_tok.size());
        put(plan.off_cbase, plan.tok.data(), sizeof(TokDev) * plan.tok.size());
        put(plan.off_comb, plan.comb.data(), sizeof(int32_t) * plan.comb.size());
        put(plan.off_tcoff, plan.tc_off.data(), sizeof(int32_t) * plan.tc_off.size());
        put(plan.off_skoff, plan.sk_off.data(), sizeof(int32_t) * plan.sk_off.size());
        memset(img + plan.off_cnt, 0, plan.desc_bytes - plan.off_cnt);
    };
    // Fused step (no rope, no host-step waves): the append takes its slots from
    // the kernel parameters and runs on the side stream while the descriptors
    // upload, instead of after them (the tiles and split-K wait for both).
    static const bool no_param_append = getenv("HG_NO_PARAM_APPEND") != nullptr;   // A/B switch
    if (tc_append && !pool->app_cnt) {
        s = cuda_check(cudaMalloc(&pool->app_cnt, 256), "cudaMalloc(append counter)");
        if (!s) s = cuda_check(cudaMemset(pool->app_cnt, 0, 256), "memset(append counter)");
        if (!s) s = cuda_check(cudaDeviceSynchronize(), "append counter init");
        if (s) { if (pool->app_cnt) cudaFree(pool->app_cnt); pool->app_cnt = nullptr; return s; }
        pool->app_total = 0;
    }
    const bool param_append = fused && !ra.rot && !pipe && !tc_append && plan.T <= kParamSlots && !no_param_append;
    // No tcgen05 items: split-K reads the new tokens' K/V from k_new / v_new, so it
    // starts at once beside the append instead of after it (the call still ends
    // after the append: st waits for it behind split-K).
    const bool sk_early = param_append && plan.tc.empty() && !plan.sk.empty();
    static const bool no_app_count = getenv("HG_TP_APPEND_JOIN") != nullptr;   // A/B: stream join instead
    if (param_append) {
        s = ensure_side(pool);
        if (!s && !pool->ev_pre) s = cuda_check(cudaEventCreateWithFlags(&pool->ev_pre, cudaEventDisableTiming), "event");
        if (!s && !pool->ev_app) s = cuda_check(cudaEventCreateWithFlags(&pool->ev_app, cudaEventDisableTiming), "event");
        if (s) return s;
        static thread_local std::vector<int64_t> slots;
        slots.resize((size_t)plan.T);
        const int B = pool->desc.block_size;
        for (int i = 0; i < v.R; ++i) {
            const int32_t *row = v.bt + (int64_t)i * v.W;
            int64_t *sl = slots.data() + plan.reqs[i].cu_q;
            for (int j = 0; j < v.n[i]; ++j) {
                const int64_t pos = (int64_t)v.c[i] + j;
                sl[j] = (int64_t)row[pos / B] * B + pos % B;
            }
        }
        s = cuda_check(cudaEventRecord(pool->ev_pre, st), "order record");   // after the caller's earlier work
        if (!s) s = cuda_check(cudaStreamWaitEvent(pool->side, pool->ev_pre, 0), "order wait");
        AttnParams bar{};   // a sharded call's peer-window entry barrier rides in this kernel
        if (outs && outs->bar_world > 0 && !sk_early) {   // (beside split-K: see below)
            for (int k = 0; k < outs->bar_world; ++k) bar.bar_flags[k] = outs->bar_flags[k];
            bar.bar_mine = outs->bar_mine;
            bar.bar_rank = outs->bar_rank;
            bar.bar_world = outs->bar_world;
            bar.bar_epoch = outs->bar_epoch;
        }
        if (outs && outs->bar_world > 0 && sk_early && !no_app_count) {
            // sharded HBM route: no stream join for the append -- it counts its CTAs in a
            // device counter and the caller's exit barrier kernel (a programmatic
            // dependent of the combine) waits for the count instead, so no event wait
            // sits between the last attention kernel and that barrier
            if (!pool->app_cnt) {
                s = cuda_check(cudaMalloc(&pool->app_cnt, 256), "cudaMalloc(append counter)");
                if (!s) s = cuda_check(cudaMemset(pool->app_cnt, 0, 256), "memset(append counter)");
                if (!s) s = cuda_check(cudaDeviceSynchronize(), "append counter init");
                if (s) { if (pool->app_cnt) cudaFree(pool->app_cnt); pool->app_cnt = nullptr; return s; }
                pool->app_total = 0;
            }
            bar.app_cnt = pool->app_cnt;
            pool->app_total += (unsigned long long)plan.T;   // one CTA per token
            outs->wait_cnt = pool->app_cnt;
            outs->wait_target = pool->app_total;
        }
        if (!s) s = launch_append_param((const uint16_t *)k_new, (const uint16_t *)v_new,
                                        (uint16_t *)pool->desc.k_cache, (uint16_t *)pool->desc.v_cache,
                                        slots.data(), plan.T, pool->desc.num_kv_heads, pool->desc.head_dim,
                                        pool->side, &bar);
        if (!s) s = cuda_check(cudaEventRecord(pool->ev_app, pool->side), "append record");
        if (s) return s;
    }
    void *dbase = nullptr;
    DescDone desc_done;
    desc_done.st = st;
    s = stage_desc(pool, build_img, plan.desc_bytes, st, &dbase, &desc_done.slot, pipe ? pipe->copy : nullptr);
    if (s) return s;
    if (param_append && !sk_early) {
        s = cuda_check(cudaStreamWaitEvent(st, pool->ev_app, 0), "append wait");
        if (s) return s;
    }
    if (pipe && pipe->enqueue_wave) {
        s = pipe->enqueue_wave(0);
        if (!s && !pipe->used) s = pipe->enqueue_wave(1);
        if (!s && !pipe->used) s = cuda_check(cudaStreamWaitEvent(st, pipe->in1, 0), "inputs wait");
        if (s) return s;
    }
    uint8_t *w = (uint8_t *)ws;
    static const bool no_sk_merge = getenv("HG_NO_SK_MERGE") != nullptr;   // A/B switch: combine kernel
    AttnParams p{};
    p.k_cache = (const uint16_t *)pool->desc.k_cache;
    p.v_cache = (const uint16_t *)pool->desc.v_cache;
    p.q = (const uint16_t *)q;
    if (outs) {
        p.n_out = outs->n;
        for (int k = 0; k < outs->n; ++k) p.outs[k] = outs->ptr[k];
        p.out_ld = outs->ld;
        if (outs->bar_world > 0) {
            if (!fused || ra.rot) return fail(HG_E_INVALID, "entry barrier needs the fused (non-rope) step");
            for (int k = 0; k < outs->bar_world; ++k) p.bar_flags[k] = outs->bar_flags[k];
            p.bar_mine = outs->bar_mine;
            p.bar_rank = outs->bar_rank;
            p.bar_world = outs->bar_world;
            p.bar_epoch = outs->bar_epoch;
        }
    } else {
        p.n_out = 1;
        p.outs[0] = (uint16_t *)out;
        p.out_ld = (int64_t)H_q * pool->desc.head_dim;
    }
    p.lse = lse;
    const uint8_t *dsc = (const uint8_t *)dbase;
    p.reqs = (const ReqDev *)(dsc + plan.off_reqs);
    p.bt_flat = (const int32_t *)(dsc + plan.off_bt);
    p.sk = (const SkItem *)(dsc + plan.off_sk);
    p.tc = (const TcItem *)(dsc + plan.off_tc);
    p.tc_tok = (const int32_t *)(dsc + plan.off_rows);
    p.tok = (const TokDev *)(dsc + plan.off_cbase);
    p.comb = (const int32_t *)(dsc + plan.off_comb);
    p.tc_off = (const int32_t *)(dsc + plan.off_tcoff);
    p.sk_off = (const int32_t *)(dsc + plan.off_skoff);
    p.sk_ctas = (int32_t)plan.sk_off.size() - 1;
    p.sk_cnt = (plan.sk_merge && !no_sk_merge) ? (unsigned int *)(dsc + plan.off_cnt) : nullptr;
    p.part_o = (float *)(w + plan.off_part_o);
    p.part_lse = (float *)(w + plan.off_part_lse);
    p.H_q = H_q;
    p.T = plan.T;
    p.n_slots = plan.n_slots;
    p.H_kv = pool->desc.num_kv_heads;
    p.G_q = H_q / p.H_kv;
    p.d = pool->desc.head_dim;
    p.n_sk = (int32_t)plan.sk.size();
    p.n_tc = (int32_t)plan.tc.size();
    p.n_comb = (int32_t)plan.comb.size();
    p.tc_ctas = plan.tc_ctas;
    p.scale_log2 = (float)(1.4426950408889634 / std::sqrt((double)p.d));
    p.trace = o ? (long long *)o->debug_trace : nullptr;
    p.sk_trace = o ? (long long *)o->debug_sk_trace : nullptr;
    if (sk_early) {
        p.k_new = (const uint16_t *)k_new;
        p.v_new = (const uint16_t *)v_new;
        // sharded: the entry barrier in split-K's first CTA (HG_TP_ENTRY_KERNEL: a 1-warp
        // kernel ahead of split-K, its programmatic primary -- A/B)
        static const bool entry_kernel = getenv("HG_TP_ENTRY_KERNEL") != nullptr;
        if (outs && outs->bar_world > 0 && !entry_kernel) {
            p.entry_word = (unsigned int *)(dsc + plan.off_exit) + 2;
        } else if (outs && outs->bar_world > 0) {
            // sharded: the peer-window entry barrier as a 1-warp kernel right ahead of
            // split-K, which is its programmatic dependent (launched at once, waiting
            // for the barrier only before its first peer-window store)
            s = launch_peer_barrier(outs->bar_flags, outs->bar_mine, outs->bar_rank, outs->bar_world,
                                    outs->bar_epoch, st, false);
            if (s) return s;
            p.bar_pdl = 1;
        }
    }
    if (tc_append) {   // the tcgen05 prologue appends; split-K reads the new keys from the inputs
        p.k_new = (const uint16_t *)k_new;
        p.v_new = (const uint16_t *)v_new;
        p.app_T = plan.T;
        p.app_bg = app_bg ? 1 : 0;
        p.app_head = app_head;
        p.app_req_cnt = pool->app_req_cnt;
        p.app_cnt = pool->app_cnt;
        pool->app_total += (unsigned long long)tc_grid;
        p.app_target = pool->app_total;
    }
    // host step with a device-visible pinned output: the rows split-K and the combine
    // finish go straight into host memory from the kernels (their PCIe writes overlap
    // the attention); the tcgen05 kernel keeps writing the device copy
    auto sk_params = [&]() {
        AttnParams q = p;
        if (pipe && pipe->zc_out) q.outs[0] = pipe->zc_out;
        return q;
    };
    int kernels = 0;
    auto rec = [&](int k, cudaStream_t on) {
        if (o && o->events[k]) cudaEventRecord((cudaEvent_t)o->events[k], on);
    };
    if (pipe && pipe->used) {
        s = ensure_side(pool);
        if (s) return s;
        s = cuda_check(cudaEventRecord(pool->ev_fork, st), "fork record");   // descriptors staged
        // wave 0 on the caller's stream: decode rows' append, then split-K
        if (!s && pipe->in0) s = cuda_check(cudaStreamWaitEvent(st, pipe->in0, 0), "wave 0 wait");
        if (!s) s = launch_append_dev(p, (const uint16_t *)k_new, (const uint16_t *)v_new, plan.T, st, 0);
        if (s) return s;
        rec(2, st);
        s = launch_splitk(sk_params(), st);
        if (s) return s;
        rec(3, st);
        // wave 1 on the pipe's stream: prefill rows' append, then the tcgen05 tiles
        if (pipe->enqueue_wave) {
            s = pipe->enqueue_wave(1);
            if (s) return s;
        }
        cudaStream_t sd = pipe->side;
        s = cuda_check(cudaStreamWaitEvent(sd, pool->ev_fork, 0), "fork wait");
        if (!s && pipe->in1) s = cuda_check(cudaStreamWaitEvent(sd, pipe->in1, 0), "wave 1 wait");
        if (!s) s = launch_append_dev(p, (const uint16_t *)k_new, (const uint16_t *)v_new, plan.T, sd, 1);
        if (s) return s;
        rec(0, sd);
        s = launch_tc(p, pool->tmap_k, pool->tmap_v, sd);
        if (s) return s;
        rec(1, sd);
        s = cuda_check(cudaEventRecord(pipe->tc_done, sd), "tc record");
        if (!s) s = cuda_check(cudaStreamWaitEvent(st, pipe->tc_done, 0), "tc wait");
        if (s) return s;
        int kernels = 4;
        if (p.n_comb && !p.sk_cnt) {   // (sk_cnt: split-K merged every partial itself)
            rec(4, st);
            s = launch_combine(sk_params(), st);
            if (s) return s;
            rec(5, st);
            ++kernels;
        } else if (p.n_comb) {   // merged in split-K: the combine events mark the kernels' joint end
            rec(4, st);
            rec(5, st);
        }
        hg_plan_stats &ls = pool->last;
        ls.tc_tiles = p.n_tc;
        ls.prefix_tiles = plan.prefix_tiles + plan.prefix_sk * p.H_kv;
        ls.splitk_items = p.n_sk * p.H_kv;
        ls.combine_rows = p.n_comb * p.H_kv;
        ls.kernels = kernels;
        ls.kv_bytes_unique = plan.kv_bytes_unique;
        ls.kv_bytes_read = plan.kv_bytes_read;
        ls.append_mode = 0;   // two-wave step: the append kernels
        return HG_OK;
    }
    // The tcgen05 tiles (tensor-bound) and the split-K items (HBM-bound) are
    // independent: the tcgen05 kernel is launched first on the caller's stream
    // (its CTAs are placed first), the split-K kernel on a side stream forked
    // after the descriptor copy; the combine waits for both.
    if (fused) {
        if (ra.rot) {   // NEXT-4: append + RoPE prologue; the attention reads the rotated Q copy
            uint16_t *q_rot = (uint16_t *)(w + plan.off_qrot);
            s = launch_rope_append_dev(p, (const uint16_t *)k_new, (const uint16_t *)v_new, (const uint16_t *)q,
                                       q_rot, plan.T, ra, st);
            p.q = q_rot;
        } else if (!param_append && !tc_append) {
            s = launch_append_dev(p, (const uint16_t *)k_new, (const uint16_t *)v_new, plan.T, st);
        }
        if (s) return s;
        if (!tc_append) ++kernels;
    }
    const bool overlap = p.n_tc && p.n_sk;
    cudaStream_t sk_stream = st;
    if (overlap) {
        s = ensure_side(pool);
        if (s) return s;
        sk_stream = pool->side;
        s = cuda_check(cudaEventRecord(pool->ev_fork, st), "fork record");
        if (s) return s;
    }
    auto do_tc = [&]() -> hg_status {
        if (!p.n_tc) return HG_OK;
        rec(0, st);
        hg_status r = launch_tc(p, pool->tmap_k, pool->tmap_v, st);
        if (r) return r;
        rec(1, st);
        ++kernels;
        return HG_OK;
    };
    auto do_sk = [&]() -> hg_status {
        if (!p.n_sk) return HG_OK;
        if (overlap) {
            hg_status r = cuda_check(cudaStreamWaitEvent(sk_stream, pool->ev_fork, 0), "fork wait");
            if (r) return r;
        }
        rec(2, sk_stream);
        hg_status r = launch_splitk(sk_params(), sk_stream);
        if (r) return r;
        rec(3, sk_stream);
        ++kernels;
        return HG_OK;
    };
    // sharded HBM route with split-K last (its partials merged in the kernel): the exit
    // barrier runs in split-K's last CTA (HG_TP_EXIT_KERNEL: its own kernel, A/B)
    static const bool exit_kernel = getenv("HG_TP_EXIT_KERNEL") != nullptr;
    const bool fold_exit = outs && outs->exit_epoch && (p.bar_pdl || p.entry_word) && !p.n_tc && p.n_sk &&
                           (!p.n_comb || p.sk_cnt) && !exit_kernel;
    if (fold_exit) {
        p.exit_epoch = outs->exit_epoch;
        p.exit_ticket = (unsigned int *)(dsc + plan.off_exit);
        p.exit_wait_cnt = outs->wait_cnt;
        p.exit_wait_target = outs->wait_target;
        outs->exit_folded = true;
    }
    if ((s = do_tc())) return s;   // first: its CTAs are placed before split-K fills the SMs
    if ((s = do_sk())) return s;
    if (overlap) {
        s = cuda_check(cudaEventRecord(pool->ev_join, sk_stream), "join record");
        if (s) return s;
        s = cuda_check(cudaStreamWaitEvent(st, pool->ev_join, 0), "join wait");
        if (s) return s;
    }
    if (p.n_comb && !p.sk_cnt) {
        rec(4, st);
        // right behind split-K on the same stream: a programmatic dependent launch
        // (resident early, waits for split-K's completion in griddepcontrol.wait)
        s = launch_combine(sk_params(), st, sk_early);
        if (s) return s;
        rec(5, st);
        ++kernels;
    } else if (p.n_comb) {   // merged in split-K: the combine events mark the kernels' joint end
        rec(4, st);
        rec(5, st);
    }
    if (sk_early && !(outs && outs->wait_cnt)) {   // the call ends after the append that ran beside split-K
        s = cuda_check(cudaStreamWaitEvent(st, pool->ev_app, 0), "append wait");
        if (s) return s;
    }
    hg_plan_stats &ls = pool->last;
    ls.tc_tiles = p.n_tc;
    ls.prefix_tiles = plan.prefix_tiles + plan.prefix_sk * p.H_kv;
    ls.splitk_items = p.n_sk * p.H_kv;   // CTAs: items x KV heads
    ls.combine_rows = p.n_comb * p.H_kv; // (token, KV head) pairs
    ls.kernels = kernels;
    ls.kv_bytes_unique = plan.kv_bytes_unique;
    ls.kv_bytes_read = plan.kv_bytes_read;
    ls.append_mode = tc_append ? (app_bg ? 2 : 1) : 0;
    return HG_OK;
}

namespace hg {
// Validate + plan once for a sharded call (pool->plan); the attention workspace bytes.
hg_status plan_attention(hg_kv_pool *pool, const hg_batch *batch, int32_t H_q, bool append, size_t *bytes,
                         const hg_attn_opts *o) {
    BatchView v;
    hg_status s = plan_call(pool, batch, H_q, o, &v, &pool->plan, append);
    if (s) return s;
    *bytes = pool->plan.total_bytes;
    return HG_OK;
}
// Attention (fused with the append when k_new != NULL) on the plan already in
// pool->plan, O to every destination of `outs` (or to `out` when outs == NULL).
hg_status attention_planned(hg_kv_pool *pool, const hg_batch *batch, int32_t H_q, const void *q,
                            const void *k_new, const void *v_new, void *out, const OutSpec *outs, void *ws,
                            size_t ws_bytes, void *stream, const hg_attn_opts *o) {
    return attention_impl(pool, batch, H_q, q, out, nullptr, ws, ws_bytes, (cudaStream_t)stream, o,
                          k_new != nullptr, k_new, v_new, outs, nullptr, true);
}
hg_status attention_to(hg_kv_pool *pool, const hg_batch *batch, int32_t H_q, const void *q, const OutSpec &outs,
                       void *ws, size_t ws_bytes, void *stream) {
    return attention_impl(pool, batch, H_q, q, nullptr, nullptr, ws, ws_bytes, (cudaStream_t)stream, nullptr, false,
                          nullptr, nullptr, &outs);
}
}  // namespace hg

extern "C" hg_status hg_hybrid_attention_ex(hg_kv_pool *pool, const hg_batch *batch, int32_t num_q_heads,
                                            const void *q, void *out, float *lse, void *workspace,
                                            size_t workspace_bytes, void *stream, const hg_attn_opts *opts) {
    if (!pool) return fail(HG_E_INVALID, "pool is NULL");
    return attention_impl(pool, batch, num_q_heads, q, out, lse, workspace, workspace_bytes,
                          (cudaStream_t)stream, opts);
}

extern "C" hg_status hg_hybrid_step(hg_kv_pool *pool, const hg_batch *batch, int32_t num_q_heads, const void *q,
                                    const void *k_new, const void *v_new, void *out, float *lse, void *workspace,
                                    size_t workspace_bytes, void *stream, const hg_attn_opts *opts) {
    if (!pool) return fail(HG_E_INVALID, "pool is NULL");
    return attention_impl(pool, batch, num_q_heads, q, out, lse, workspace, workspace_bytes, (cudaStream_t)stream,
                          opts, true, k_new, v_new);
}

extern "C" hg_status hg_hybrid_attention(hg_kv_pool *pool, const hg_batch *batch, int32_t num_q_heads,
                                         const void *q, void *out, float *lse, void *workspace,
                                         size_t workspace_bytes, void *stream) {
    return hg_hybrid_attention_ex(pool, batch, num_q_heads, q, out, lse, workspace, workspace_bytes, stream,
                                  nullptr);
}

extern "C" hg_status hg_plan_rows(const hg_batch *batch, int32_t H_q, int32_t H_kv, int32_t d, int32_t num_blocks,
                                  int32_t num_sms, int32_t use_tc, const hg_attn_opts *o, hg_plan_row *rows,
                                  int64_t cap, int64_t *n_rows) {
    if (!n_rows || (cap > 0 && !rows) || num_sms < 1) return fail(HG_E_INVALID, "bad arguments");
    BatchView v;
    hg_status s = view_batch(batch, &v);
    if (s) return s;
    s = validate(v, kBlock, num_blocks, H_q, H_kv, false);
    if (s) return s;
    PlanOpts po;
    po.num_sms = num_sms;
    if (o) {
        po.split_tokens = o->split_tokens;
        po.prefix_pass = !o->disable_prefix_pass;
        po.split_prefill = !o->disable_prefill_split;
        po.route = o->route;
        if (o->disable_tc) use_tc = 0;
    }
    po.use_tc = use_tc != 0;
    static thread_local Plan plan;
    s = build_plan(v, H_q, H_kv, d, po, &plan);
    if (s) return s;
    const int G = H_q / H_kv;
    int64_t n = 0;
    auto emit = [&](int t, int h, int k0, int k1, int part, int kind) {
        if (n < cap) rows[n] = hg_plan_row{t, h, k0, k1, part, kind, plan.tok[t].nparts};
        ++n;
    };
    for (const TcItem &it : plan.tc)
        for (int r = 0; r < it.nrows; ++r) {
            const int x = it.hl0 + r, j = x / G, h = it.g * G + x % G;
            if (it.mode == 0) emit(it.t0 + j, h, it.k0, std::min(it.k1, it.pos0 + j + 1), it.part, 0);
            else emit(plan.tc_tok[it.t0 + j], h, it.k0, it.k1, it.part, 1);
        }
    for (const SkItem &it : plan.sk) {
        const ReqDev &rq = plan.reqs[it.req];
        for (int g = 0; g < H_kv; ++g)
            for (int r = 0; r < it.nrows; ++r) {   // the rows the kernel computes (SkItem stacking)
                const int x = it.hl0 + r, j = it.j0 + x / G;
                if (it.mode) emit(plan.tc_tok[j], g * G + x % G, it.k0, it.k1, it.part, 3);   // prefix node
                else emit(rq.cu_q + j, g * G + x % G, it.k0, std::min(it.k1, rq.c + j + 1), it.part, 2);
            }
    }
    *n_rows = n;
    return HG_OK;
}

extern "C" hg_status hg_last_plan_stats(const hg_kv_pool *pool, hg_plan_stats *out) {
    if (!pool || !out) return fail(HG_E_INVALID, "NULL argument");
    *out = pool->last;
    return HG_OK;
}

// ---------------------------------------------------------------------------
// e2e step with host buffers
// ---------------------------------------------------------------------------
static size_t al256(size_t x) { return (x + 255) / 256 * 256; }

// The host step's plan options: with both prefill chunks and decode rows, the
// prefill chunks on tcgen05 tiles (they consume the second input wave on their own
// stream while split-K runs on the first, which hides most of the PCIe upload;
// the HBM route would put both waves' rows into one split-K launch behind the
// whole upload) and shared-prefix nodes on split-K (route 3), so split-K merges
// every decode row's partials itself and its final rows leave as it runs.
static hg_attn_opts host_step_opts(const BatchView &v) {
    bool has_pre = false, has_dec = false;
    for (int i = 0; i < v.R; ++i) (v.n[i] > 1 ? has_pre : has_dec) = true;
    hg_attn_opts ho{};
    static const bool nodes_tc = getenv("HG_E2E_NODES_TC") != nullptr;   // A/B: prefix nodes on tcgen05 (route 1)
    ho.route = has_pre && has_dec ? (nodes_tc ? 1 : 3) : 0;
    return ho;
}

static bool device_visible_host(const void *p) {
    cudaPointerAttributes pa{};
    const bool ok = cudaPointerGetAttributes(&pa, p) == cudaSuccess && pa.type == cudaMemoryTypeHost && pa.devicePointer;
    cudaGetLastError();
    return ok;
}

extern "C" hg_status hg_hybrid_step_host_workspace_size(const hg_kv_pool *pool, const hg_batch *batch,
                                                        int32_t H_q, size_t *bytes) {
    if (!pool || !bytes) return fail(HG_E_INVALID, "NULL argument");
    BatchView v;
    hg_status s = view_batch(batch, &v);
    if (s) return s;
    const hg_attn_opts ho = host_step_opts(v);
    Plan plan;
    s = plan_call(const_cast<hg_kv_pool *>(pool), batch, H_q, &ho, &v, &plan, true);
    if (s) return s;
    const size_t attn = plan.total_bytes;
    int64_t T = 0;
    for (int i = 0; i < batch->num_reqs; ++i) T += batch->new_len[i];
    const size_t d = pool->desc.head_dim, Hk = pool->desc.num_kv_heads;
    *bytes = 2 * al256(T * H_q * d * 2) + 2 * al256(T * Hk * d * 2) + al256(T * 8) + al256(attn);
    return HG_OK;
}

// Pipelined: the inputs go up in two waves on a library-owned copy stream, the
// decode rows' first (small: one token per request) so the HBM-bound split-K
// kernel starts after ~1/10 of the upload; the prefill chunks' rows follow while
// it runs and feed the tcgen05 tiles on a high-priority stream; their O goes
// back to the host as soon as those tiles finish, the decode rows' after the
// combine.  Runs of consecutive requests of one wave are copied as one range.
static hg_status step_host_impl(hg_kv_pool *pool, const hg_batch *batch, int32_t H_q, const void *q_host,
                                const void *k_new_host, const void *v_new_host, void *out_host, void *workspace,
                                size_t workspace_bytes, void *stream, bool sync);

extern "C" hg_status hg_hybrid_step_host(hg_kv_pool *pool, const hg_batch *batch, int32_t H_q,
                                         const void *q_host, const void *k_new_host, const void *v_new_host,
                                         void *out_host, void *workspace, size_t workspace_bytes, void *stream) {
    return step_host_impl(pool, batch, H_q, q_host, k_new_host, v_new_host, out_host, workspace, workspace_bytes,
                          stream, true);
}

extern "C" hg_status hg_hybrid_step_host_async(hg_kv_pool *pool, const hg_batch *batch, int32_t H_q,
                                               const void *q_host, const void *k_new_host, const void *v_new_host,
                                               void *out_host, void *workspace, size_t workspace_bytes,
                                               void *stream) {
    return step_host_impl(pool, batch, H_q, q_host, k_new_host, v_new_host, out_host, workspace, workspace_bytes,
                          stream, false);
}

// Cheap identity of a batch for the plan-ahead: its pointers, shape and per-request
// lengths (not the block-table contents -- the caller keeps those unchanged).
static uint64_t batch_fingerprint(const BatchView &v, const hg_batch *b) {
    uint64_t h = 1469598103934665603ull;
    auto mix = [&](uint64_t x) { h = (h ^ x) * 1099511628211ull; };
    mix((uint64_t)(uintptr_t)b);
    mix((uint64_t)(uintptr_t)v.bt);
    mix((uint64_t)v.R);
    mix((uint64_t)v.W);
    for (int i = 0; i < v.R; ++i) mix(((uint64_t)(uint32_t)v.c[i] << 32) ^ ((uint64_t)(uint32_t)v.n[i] << 8) ^ (uint32_t)v.s[i]);
    return h;
}

extern "C" hg_status hg_hybrid_step_host_plan(hg_kv_pool *pool, const hg_batch *batch, int32_t H_q) {
    if (!pool || !batch) return fail(HG_E_INVALID, "NULL argument");
    pool->ahead_ok = false;
    BatchView v;
    hg_status s = view_batch(batch, &v);
    if (s) return s;
    const hg_attn_opts ho = host_step_opts(v);
    s = plan_call(pool, batch, H_q, &ho, &v, &pool->plan_ahead, true);
    if (s) return s;
    pool->ahead_ok = true;
    pool->ahead_batch = batch;
    pool->ahead_Hq = H_q;
    pool->ahead_fp = batch_fingerprint(v, batch);
    return HG_OK;
}

static hg_status step_host_impl(hg_kv_pool *pool, const hg_batch *batch, int32_t H_q, const void *q_host,
                                const void *k_new_host, const void *v_new_host, void *out_host, void *workspace,
                                size_t workspace_bytes, void *stream, bool sync) {
    static const bool trace = getenv("HG_E2E_TRACE") != nullptr;   // host-side phase times (stderr)
    auto now = [] { return std::chrono::steady_clock::now(); };
    auto us = [](std::chrono::steady_clock::time_point a, std::chrono::steady_clock::time_point b) {
        return std::chrono::duration<double, std::micro>(b - a).count();
    };
    const auto t_in = now();
    if (!pool) return fail(HG_E_INVALID, "pool is NULL");
    hg_status s = sticky_check();
    if (s) return s;
    if (!q_host || !k_new_host || !v_new_host || !out_host) return fail(HG_E_INVALID, "host buffer NULL");
    BatchView v;
    s = view_batch(batch, &v);
    if (s) return s;
    // Workspace: the device copies of q, out, k_new, v_new first (sized by T
    // alone), then the attention workspace -- so wave 0's copies can start
    // before the batch is validated and planned.
    int64_t T = 0;
    bool rows_ok = true;
    for (int i = 0; i < v.R; ++i) {
        rows_ok &= v.n[i] >= 1;
        T += v.n[i];
    }
    const size_t d = pool->desc.head_dim, Hk = pool->desc.num_kv_heads;
    const size_t qrow = (size_t)std::max(H_q, 0) * d * 2, kvrow = Hk * d * 2;   // bytes per token row
    const size_t in_bytes = rows_ok ? 2 * al256(T * qrow) + 2 * al256(T * kvrow) + al256(T * 8) : 0;
    uint8_t *w = (uint8_t *)workspace;
    uint8_t *q_d = w, *o_d = q_d + al256(T * qrow), *k_d = o_d + al256(T * qrow), *v_d = k_d + al256(T * kvrow);
    cudaStream_t st = (cudaStream_t)stream;
    s = ensure_hi(pool);
    if (s) return s;
    if (!pool->h2d) {
        s = cuda_check(cudaStreamCreateWithFlags(&pool->h2d, cudaStreamNonBlocking), "copy stream");
        for (cudaEvent_t *e : {&pool->ev_in0, &pool->ev_in1, &pool->ev_d2h})
            if (!s) s = cuda_check(cudaEventCreateWithFlags(e, cudaEventDisableTiming), "event create");
        if (s) return s;
    }
    // row runs [a, b) of each wave (wave 1 = prefill-chunk requests, n_i > 1)
    std::vector<std::pair<int64_t, int64_t>> runs[2];
    if (rows_ok) {
        int64_t row = 0;
        for (int i = 0; i < v.R; ++i) {
            auto &rw = runs[v.n[i] > 1 ? 1 : 0];
            if (!rw.empty() && rw.back().second == row) rw.back().second += v.n[i];
            else rw.emplace_back(row, row + v.n[i]);
            row += v.n[i];
        }
    }
    bool issued[2] = {false, false};
    auto enqueue_wave = [&](int wv) -> hg_status {
        if (issued[wv]) return HG_OK;
        issued[wv] = true;
        for (auto &r : runs[wv]) {
            const int64_t a = r.first, n = r.second - r.first;
            hg_status e = cuda_check(cudaMemcpyAsync(q_d + a * qrow, (const uint8_t *)q_host + a * qrow, n * qrow,
                                                     cudaMemcpyHostToDevice, pool->h2d), "H2D q");
            if (!e) e = cuda_check(cudaMemcpyAsync(k_d + a * kvrow, (const uint8_t *)k_new_host + a * kvrow,
                                                   n * kvrow, cudaMemcpyHostToDevice, pool->h2d), "H2D k");
            if (!e) e = cuda_check(cudaMemcpyAsync(v_d + a * kvrow, (const uint8_t *)v_new_host + a * kvrow,
                                                   n * kvrow, cudaMemcpyHostToDevice, pool->h2d), "H2D v");
            if (e) return e;
        }
        return cuda_check(cudaEventRecord(wv ? pool->ev_in1 : pool->ev_in0, pool->h2d), "wave record");
    };
    // the copy stream and the tcgen05 stream start after whatever the caller queued before this step
    s = cuda_check(cudaEventRecord(pool->ev_d2h, st), "order record");
    if (!s) s = cuda_check(cudaStreamWaitEvent(pool->h2d, pool->ev_d2h, 0), "order wait");
    if (!s) s = cuda_check(cudaStreamWaitEvent(pool->side_hi, pool->ev_d2h, 0), "order wait");
    if (s) return s;
    const bool early = rows_ok && T > 0 && workspace && workspace_bytes >= in_bytes;
    if (early) {   // wave 0 (decode rows, small) crosses PCIe while the host validates and plans
        s = enqueue_wave(0);
        if (s) return s;
    }
    // on any error below, the copies already queued finish before returning (they
    // read the caller's host buffers); nothing else has been launched
    auto bail = [&](hg_status e) {
        if (early) cudaStreamSynchronize(pool->h2d);
        return e;
    };
    // one validated plan for the whole step (attention_impl reuses pool->plan)
    static const bool no_zc = getenv("HG_E2E_NO_ZC") != nullptr;   // A/B: copy every row back
    const bool pinned_out = !no_zc && device_visible_host(out_host);
    const hg_attn_opts ho = host_step_opts(v);
    if (pool->ahead_ok && pool->ahead_batch == batch && pool->ahead_Hq == H_q &&
        pool->ahead_fp == batch_fingerprint(v, batch)) {
        std::swap(pool->plan, pool->plan_ahead);   // planned while the previous step ran
    } else {
        s = plan_call(pool, batch, H_q, &ho, &v, &pool->plan, true);
    }
    pool->ahead_ok = false;
    if (s) return bail(s);
    if (T == 0) return HG_OK;
    const size_t attn = pool->plan.total_bytes;
    const size_t need = in_bytes + al256(attn);
    if (!workspace || workspace_bytes < need)
        return bail(fail(HG_E_INVALID, "workspace too small (%zu < %zu)", workspace_bytes, need));
    uint8_t *ws_attn = w + in_bytes;
    // Zero-copy result: when out_host is pinned, device-visible host memory, the rows
    // written by split-K / the combine (every row on the HBM route, the decode rows on
    // the tcgen05 route) are stored there by the kernels, and only the tcgen05 kernel's
    // rows are copied back -- unless a prefill chunk is cut into key ranges (its rows
    // then come from the combine after the tcgen05 copy-back was planned)
    uint16_t *zc = nullptr;
    if (pinned_out) {
        cudaPointerAttributes pa{};
        bool cut = false;
        for (size_t k = 0; !cut && k < pool->plan.tok.size(); ++k)
            cut = v.n[pool->plan.tok[k].req] > 1 && pool->plan.tok[k].nparts > 1 && !pool->plan.tc.empty();
        if (!cut && cudaPointerGetAttributes(&pa, out_host) == cudaSuccess) zc = (uint16_t *)pa.devicePointer;
        cudaGetLastError();
    }
    StepPipe pipe;
    pipe.zc_out = zc;
    pipe.copy = pool->h2d;
    pipe.in0 = pool->ev_in0;
    pipe.in1 = pool->ev_in1;
    pipe.side = pool->side_hi;
    pipe.tc_done = pool->ev_tc;
    pipe.planned = true;
    pipe.enqueue_wave = enqueue_wave;
    const auto t_cp = now();
    s = attention_impl(pool, batch, H_q, q_d, o_d, nullptr, ws_attn, attn, st, nullptr, true, k_d, v_d, nullptr,
                       &pipe);
    if (s) return bail(s);
    const auto t_at = now();
    auto d2h = [&](const std::vector<std::pair<int64_t, int64_t>> &rw, cudaStream_t on) -> hg_status {
        for (auto &r : rw) {
            hg_status e = cuda_check(cudaMemcpyAsync((uint8_t *)out_host + r.first * qrow, o_d + r.first * qrow,
                                                     (r.second - r.first) * qrow, cudaMemcpyDeviceToHost, on), "D2H out");
            if (e) return e;
        }
        return HG_OK;
    };
    // Prefill rows are final when the tcgen05 kernel ends -- unless the planner
    // cut a chunk's keys into ranges (partials merged by the combine kernel on
    // the caller's stream): then they are read back after the combine too.
    bool prefill_cut = false;
    for (size_t k = 0; pipe.used && !prefill_cut && k < pool->plan.tok.size(); ++k)
        prefill_cut = v.n[pool->plan.tok[k].req] > 1 && pool->plan.tok[k].nparts > 1;
    if (pipe.used && prefill_cut) {
        s = cuda_check(cudaMemcpyAsync(out_host, o_d, T * qrow, cudaMemcpyDeviceToHost, st), "D2H out");
    } else if (pipe.used) {
        s = d2h(runs[1], pipe.side);
        if (!s) s = cuda_check(cudaEventRecord(pool->ev_d2h, pipe.side), "d2h record");
        if (!s && !pipe.zc_out) s = d2h(runs[0], st);   // zero-copy: split-K / the combine wrote them
        if (!s) s = cuda_check(cudaStreamWaitEvent(st, pool->ev_d2h, 0), "d2h wait");
    } else if (!pipe.zc_out) {
        s = cuda_check(cudaMemcpyAsync(out_host, o_d, T * qrow, cudaMemcpyDeviceToHost, st), "D2H out");
    }   // else zero-copy: every row came from split-K / the combine
    if (s) return s;
    const auto t_d2 = now();
    if (!sync) return HG_OK;   // hg_hybrid_step_host_async: the caller synchronises `stream`
    s = cuda_check(cudaStreamSynchronize(st), "stream sync");
    if (trace)
        fprintf(stderr, "hg_hybrid_step_host: prep %.1f us, attention + input copies enqueue %.1f, d2h %.1f, sync %.1f\n",
                us(t_in, t_cp), us(t_cp, t_at), us(t_at, t_d2), us(t_d2, now()));
    return s;
}

// ---------------------------------------------------------------------------
// a.9 predictor: features, OLS (Householder QR), predict
// ---------------------------------------------------------------------------
extern "C" hg_status hg_batch_features(const hg_batch *batch, int32_t block_size, hg_features *out) {
    if (!out || block_size < 1) return fail(HG_E_INVALID, "bad arguments");
    BatchView v;
    hg_status s = view_batch(batch, &v);
    if (s) return s;
    hg_features f{};
    // D_ctx = unique KV slots read by decode rows (R15): a slot of a physically
    // shared block is counted once however many decode rows (at whatever prefix
    // depth) see it; a row sees positions [0, c_i] of its table.
    static thread_local std::vector<std::pair<int32_t, int32_t>> seen;  // (shared id, slots visible)
    seen.clear();
    for (int i = 0; i < v.R; ++i) {
        const int64_t c = v.c[i], n = v.n[i];
        if (n == 1 && c >= 1) {
            f.N_d += 1;
            f.S_d += 1;
            const int64_t s_tok = std::min<int64_t>((int64_t)v.s[i] * block_size, c + 1);
            f.D_ctx += (double)(c + 1 - s_tok);
            const int32_t *row = v.bt + (int64_t)i * v.W;
            for (int64_t k = 0; k * block_size < s_tok; ++k)
                seen.push_back({row[k], (int32_t)std::min<int64_t>(block_size, s_tok - k * block_size)});
        } else {
            f.N_p += 1;
            f.S_p += (double)n;
            f.P2 += (double)n * ((double)c + (double)(n + 1) / 2.0);
        }
    }
    std::sort(seen.begin(), seen.end());
    for (size_t k = 0; k < seen.size(); ++k)   // the largest visible count per id (last of its run)
        if (k + 1 == seen.size() || seen[k + 1].first != seen[k].first) f.D_ctx += (double)seen[k].second;
    f.S_p2 = f.S_p * f.S_p;
    f.S_d2 = f.S_d * f.S_d;
    *out = f;
    return HG_OK;
}

static void feat_vec(const hg_features &f, double x[8]) {
    x[0] = f.S_p; x[1] = f.S_d; x[2] = f.S_p2; x[3] = f.S_d2;
    x[4] = f.N_p; x[5] = f.N_d; x[6] = f.P2; x[7] = f.D_ctx;
}

extern "C" hg_status hg_predictor_fit(const hg_features *X, const double *y, int32_t n, int32_t mask,
                                      hg_predictor *out) {
    if (!X || !y || !out || n < 1 || (mask & ~0x1FF)) return fail(HG_E_INVALID, "bad arguments");
    const bool rel = mask & HG_FIT_RELATIVE;
    if (rel)
        for (int i = 0; i < n; ++i)
            if (!(y[i] > 0)) return fail(HG_E_INVALID, "HG_FIT_RELATIVE needs y > 0 (y[%d] = %g)", i, y[i]);
    int cols[8], k = 0;
    for (int b = 0; b < 8; ++b)
        if (mask >> b & 1) cols[k++] = b;
    const int p = k + 1;
    if (n < p) return fail(HG_E_RANK_DEFICIENT, "%d samples < %d parameters", n, p);
    // A = [1, x_cols] scaled column-wise by max |.| (conditioning), column-major
    std::vector<double> A((size_t)n * p), b(y, y + n), scale(p, 1.0);
    for (int i = 0; i < n; ++i) {
        double x[8];
        feat_vec(X[i], x);
        A[i] = 1.0;
        for (int j = 0; j < k; ++j) A[(size_t)(j + 1) * n + i] = x[cols[j]];
        if (rel) {   // row i weighted by 1 / y_i: residual (w.x_i - y_i) / y_i
            for (int j = 0; j < p; ++j) A[(size_t)j * n + i] /= y[i];
            b[i] = 1.0;
        }
    }
    for (int j = 0; j < p; ++j) {
        double m = 0;
        for (int i = 0; i < n; ++i) m = std::max(m, std::fabs(A[(size_t)j * n + i]));
        if (m == 0) return fail(HG_E_RANK_DEFICIENT, "feature column %d is identically zero", j);
        scale[j] = m;
        for (int i = 0; i < n; ++i) A[(size_t)j * n + i] /= m;
    }
    // Householder QR, applying reflections to b
    std::vector<double> diag(p);
    double rmax = 0;
    for (int j = 0; j < p; ++j) {
        double *aj = &A[(size_t)j * n];
        double norm = 0;
        for (int i = j; i < n; ++i) norm += aj[i] * aj[i];
        norm = std::sqrt(norm);
        double alpha = aj[j] > 0 ? -norm : norm;
        diag[j] = alpha;
        rmax = std::max(rmax, std::fabs(alpha));
        if (std::fabs(alpha) <= 1e-12 * std::max(rmax, 1.0))
            return fail(HG_E_RANK_DEFICIENT, "design matrix is rank deficient at column %d (mask 0x%x)", j, mask);
        aj[j] -= alpha;  // v = a - alpha e_j
        double vnorm2 = 0;
        for (int i = j; i < n; ++i) vnorm2 += aj[i] * aj[i];
        auto reflect = [&](double *c) {
            double dot = 0;
            for (int i = j; i < n; ++i) dot += aj[i] * c[i];
            double f = 2.0 * dot / vnorm2;
            for (int i = j; i < n; ++i) c[i] -= f * aj[i];
        };
        for (int jj = j + 1; jj < p; ++jj) reflect(&A[(size_t)jj * n]);
        reflect(b.data());
    }
    // back substitution R w = Q^T b (R upper: diag[j] on the diagonal, A above)
    std::vector<double> w(p);
    for (int j = p - 1; j >= 0; --j) {
        double acc = b[j];
        for (int jj = j + 1; jj < p; ++jj) acc -= A[(size_t)jj * n + j] * w[jj];
        w[j] = acc / diag[j];
    }
    hg_predictor m{};
    m.w[0] = w[0] / scale[0];
    for (int j = 0; j < k; ++j) m.w[1 + cols[j]] = w[j + 1] / scale[j + 1];
    m.feature_mask = mask;
    m.n_samples = n;
    double err = 0;
    for (int i = 0; i < n; ++i) err += std::fabs(hg_predictor_predict(&m, &X[i]) - y[i]) / y[i];
    m.train_mape = err / n;
    *out = m;
    return HG_OK;
}

extern "C" double hg_predictor_predict(const hg_predictor *m, const hg_features *f) {
    if (!m || !f) return 0.0;
    double x[8];
    feat_vec(*f, x);
    double acc = m->w[0];
    for (int k = 0; k < 8; ++k) acc += m->w[1 + k] * x[k];
    return acc > 0 ? acc : 0.0;
}

namespace hg {
int pool_num_kv_heads(const hg_kv_pool *p) { return p->desc.num_kv_heads; }
int pool_head_dim(const hg_kv_pool *p) { return p->desc.head_dim; }
}  // namespace hg
