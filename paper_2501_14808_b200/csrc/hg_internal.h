// hg_internal.h -- structures shared by the host planner (host.cpp / api.cpp)
// and the sm_100a kernels (kernels.cu, tc_attn.cu).  Not part of the C ABI.
#pragma once
#include <cstdint>
#include <cstddef>
#include <string>
#include <vector>

#include "hygen.h"

// Device-side invariant checks (index ranges, arrival counts): compiled in only for the
// checking build (HG_NVCC_DEFS=-DHG_CHECKS, tools/gpurun/r2_checks.sh) -- a failed check
// prints its condition and traps (sticky HG_E_CUDA), so parity tests fail on it.
#ifdef HG_CHECKS
#define HG_DCHECK(c)                                                                           \
    do {                                                                                       \
        if (!(c)) {                                                                            \
            printf("HG_DCHECK failed %s:%d: %s\n", __FILE__, __LINE__, #c);                   \
            __trap();                                                                          \
        }                                                                                      \
    } while (0)
#else
#define HG_DCHECK(c) \
    do {             \
    } while (0)
#endif

namespace hg {

constexpr int kBlock = 16;        // KV block size B handled by the kernels
constexpr int kSkRows = 16;       // query rows per split-K item (one m16 MMA tile)
constexpr int kTcRows = 128;      // query rows per tcgen05 tile (UMMA M)
constexpr int kTcKeys = 128;      // keys per tcgen05 KV tile (UMMA N of S = Q K^T)
constexpr int kMaxCuts = 64;      // key ranges per prefill request (build_plan)
constexpr int kMaxOuts = 8;       // O copies one launch writes (ranks of a peer window)

// Per-request record in the device descriptor.
struct ReqDev {
    int32_t c;       // cached length c_i
    int32_t n;       // new tokens n_i
    int32_t cu_q;    // first batch row of the request
    int32_t bt_off;  // offset of the request's block ids in bt_flat
    // background append of a fused tcgen05 step (AttnParams.app_bg): the next request
    // in need order (-1: last), and the count app_req_cnt[i] reaches once every
    // CTA has written its slice of this request's new tokens
    int32_t app_next = -1;
    int32_t pad_ = 0;
    unsigned long long app_tgt = 0;
};

// Split-K item (sm_100a mma.sync path, kernels.cu), launched once per KV head g
// (grid.y): up to 16 stacked query rows of one request against keys [k0, k1)
// further capped per row by causality.  Stacked row r has index x = hl0 + r:
// token j0 + x / G_q, q head g*G_q + x % G_q.  G_q <= 16: hl0 = 0 and the item
// stacks nt whole tokens (nt * G_q <= 16); G_q > 16: one token per item, its
// q heads cut into ceil(G_q / 16) items of <= 16 rows (hl0 = 0, 16, ...).
struct SkItem {
    int32_t req;
    int32_t j0;
    int32_t nt;     // tokens the item touches
    int32_t k0;     // multiple of kBlock
    int32_t k1;
    int32_t part;   // partial index for rows that are combined (-1: direct write)
    int32_t hl0;    // stacked-row offset inside token j0 (q-head-in-group of row 0)
    int32_t nrows;  // stacked rows (<= kSkRows)
    int32_t mode;   // 0: rows of request `req` (causal); 1: prefix node -- member x / G_q is token
                    // tc_tok[j0 + x / G_q], every row sees all of [k0, k1); `req` gives the block table
};

// Per batch token: where its partials live.  Partial slot of (token t, KV head
// g, part, q-head-in-group hl) = base + (g * nparts + part) * G_q + hl;
// base = -1 means the token's rows have one part and are written directly.
struct TokDev {
    int32_t base;
    int32_t nparts;
    int32_t req;    // owning request (device-side slot computation of the fused append)
    int32_t wave;   // pipelined host step: input wave of the token (0 decode rows, 1 prefill-chunk rows)
};

// tcgen05 tile (tc_attn.cu): up to 128 stacked query rows sharing KV head g
// and a key range [k0, k1) of ONE block table (the request's, or the group
// prefix's).  Stacked row r has index x = hl0 + r, token slot j = x / G_q and
// q head g*G_q + x % G_q:
//   mode 0 (prefill chunk): token t = t0 + j, causal limit pos0 + j + 1
//   mode 1 (prefix group):  token t = tc_tok[t0 + j] (member decode rows), limit k1
struct TcItem {
    int32_t bt_off;  // block table (bt_flat offset) the keys are read through
    int32_t g;
    int32_t k0;      // multiple of kBlock (0 for mode 0)
    int32_t k1;
    int32_t mode;
    int32_t t0;
    int32_t nrows;   // <= 128
    int32_t part;    // partial index (-1: rows written directly)
    int32_t pos0;    // mode 0: absolute position of token t0
    int32_t hl0;     // q-head-in-group of stacked row 0
    int32_t cnew;    // first key position written by this call (c_i of the request; INT32_MAX: none)
};

// Device-side view of one attention call.
struct AttnParams {
    const uint16_t *k_cache;
    const uint16_t *v_cache;
    const uint16_t *q;
    // O destinations: element (t, h, :) of every copy lives at outs[k] + t*out_ld + h*d.
    // One copy on a single GPU; under KV-head sharding with a peer window, one per
    // rank (NVLink peer pointers, already offset to this rank's head slice), so the
    // epilogues do the all-gather themselves.
    uint16_t *outs[kMaxOuts];
    int32_t n_out;
    int64_t out_ld;
    float *lse;
    const ReqDev *reqs;
    const int32_t *bt_flat;
    const SkItem *sk;
    const TcItem *tc;
    const int32_t *tc_tok;     // member tokens of prefix-group tiles
    const TokDev *tok;         // [T]
    const int32_t *comb;       // tokens whose rows are merged (combine grid.x)
    float *part_o;             // [slots][d] normalised partial outputs
    float *part_lse;           // [slots] log2-domain LSE of each partial (-inf: empty)
    int32_t H_q, H_kv, G_q, d;
    int32_t T;                 // batch tokens (rows of q / O)
    int64_t n_slots;           // partial slots in part_o / part_lse
    int32_t n_sk, n_tc, n_comb;
    int32_t tc_ctas;           // persistent tcgen05 grid (<= n_tc)
    const int32_t *tc_off;     // [tc_ctas + 1]: CTA b processes tc items [tc_off[b], tc_off[b+1])
    int32_t sk_ctas;           // persistent split-K grid per KV head (grid = sk_ctas x H_kv)
    const int32_t *sk_off;     // [sk_ctas + 1]: CTA b processes split-K items [sk_off[b], sk_off[b+1])
    float scale_log2;          // log2(e) / sqrt(d)
    // peer-window entry barrier folded into the fused step's append kernel (bar_world = 0: none)
    unsigned long long *bar_flags[kMaxOuts];
    unsigned long long *bar_mine;
    int32_t bar_rank, bar_world;
    unsigned long long bar_epoch;
    long long *trace;          // debug: per-event clock64 stamps of tcgen05 CTA 0 (NULL: off)
    long long *sk_trace;       // debug: %globaltimer at each split-K CTA's start / end (NULL: off)
    // Fused step with the append running beside split-K (no tcgen05 items): split-K
    // reads the new tokens' K/V (positions [c_i, c_i + n_i)) from these inputs
    // instead of the cache the append is still writing (NULL: everything from the cache).
    const uint16_t *k_new, *v_new;
    // ... and, in a sharded call, split-K is a programmatic dependent of the
    // peer-window entry barrier kernel: it waits for that grid (griddepcontrol.wait)
    // before its first peer-window store and before it completes.
    int32_t bar_pdl;
    // Fused step on the tcgen05 route: the tcgen05 CTAs append this call's K/V
    // (k_new / v_new, app_T tokens, split evenly over the grid) in their prologue
    // and count themselves in app_cnt; a TMA producer waits for app_cnt >=
    // app_target (every share written) before the first tile holding a new key.
    // app_T = 0: the append ran as its own kernel before.
    unsigned long long *app_cnt;
    unsigned long long app_target;
    int32_t app_T;
    // app_bg = 1: written in the background by each CTA's idle warp 11, request by
    // request in need order (the list from app_head through ReqDev.app_next, each
    // request's tokens sliced over the grid, app_req_cnt[i] counting the slices
    // done); a TMA producer waits for its item's request only.  0: all 384 threads
    // append the CTA's share before the pipelines start (global count app_cnt).
    int32_t app_bg;
    int32_t app_head;
    unsigned long long *app_req_cnt;
    // In-kernel merge (no tcgen05 items, so every partial comes from split-K):
    // arrival counters [T][H_kv], zero in every call's descriptor image; the split-K
    // CTA completing a token's partials merges its rows and no combine kernel runs.
    // NULL: partials are merged by combine_kernel.
    unsigned int *sk_cnt;
    // Sharded HBM route with split-K as the call's last kernel: the peer-window exit
    // barrier runs in split-K's last CTA (exit_ticket counts finished CTAs, zero in
    // the descriptor image) instead of a kernel of its own; it waits for the side-
    // stream append's count first.  exit_epoch = 0: no folded barrier.
    // sharded HBM route: split-K's first CTA runs the entry barrier (bar_* fields);
    // entry_word[0] its ticket, [1] set once through (desc image, zero each call; NULL: none)
    unsigned int *entry_word;
    unsigned long long exit_epoch;
    unsigned int *exit_ticket;
    const unsigned long long *exit_wait_cnt;
    unsigned long long exit_wait_target;
};

// Host-side plan (a.1 + a.4): built per call, staged to the device.
struct Plan {
    int R = 0, T = 0, W = 0;
    std::vector<ReqDev> reqs;
    int64_t n_bt = 0;                // flattened block ids (request i's at ReqDev.bt_off)
    std::vector<SkItem> sk;
    std::vector<TcItem> tc;
    std::vector<int32_t> tc_tok;
    std::vector<SkItem> sk_tmp;
    std::vector<TcItem> tc_tmp;
    std::vector<int32_t> tc_off;   // per-CTA item ranges of the persistent tcgen05 grid
    std::vector<int32_t> sk_off;   // per-CTA item ranges of the persistent split-K grid (per KV head)
    std::vector<TokDev> tok;
    std::vector<int32_t> comb;
    int64_t n_slots = 0;
    int32_t prefix_tiles = 0;   // tcgen05 prefix-node tiles (tcgen05 route)
    int32_t prefix_sk = 0;      // prefix-node split-K items (HBM route; one CTA per KV head each)
    int64_t n_tc_prefill() const { return (int64_t)tc.size() - prefix_tiles; }   // mode-0 items
    int64_t kv_bytes_unique = 0;
    int64_t kv_bytes_read = 0;
    int32_t tc_ctas = 0;        // persistent tcgen05 grid chosen by the planner
    bool sk_merge = false;      // partials merged inside split-K (AttnParams.sk_cnt)
    // device layout (byte offsets inside the workspace)
    size_t off_reqs = 0, off_bt = 0, off_sk = 0, off_tc = 0, off_rows = 0, off_cbase = 0,
           off_comb = 0, off_tcoff = 0, off_skoff = 0, off_cnt = 0, off_exit = 0, off_qrot = 0, desc_bytes = 0, off_part_o = 0, off_part_lse = 0, total_bytes = 0;
};

// ---- host helpers (host.cpp) ------------------------------------------------
void set_error(const char *fmt, ...);
hg_status fail(hg_status s, const char *fmt, ...);

struct BatchView {
    int R, W;
    const int32_t *bt, *c, *n, *s;
    std::vector<int32_t> s_store;  // zeros when shared_prefix_blocks == NULL
};
hg_status view_batch(const hg_batch *b, BatchView *v);
// Validation rules of SURVEY §8(b); num_q_heads < 0 skips the head check.
hg_status validate(const BatchView &v, int block_size, int num_blocks, int num_q_heads, int H_kv,
                   bool append);
void prefix_groups(const BatchView &v, std::vector<int32_t> *group);

struct KernelEvents {
    void *ev[6] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
};

struct PlanOpts {
    int split_tokens = 0;
    bool prefix_pass = true;
    bool use_tc = true;
    bool split_prefill = true;   // key-range cuts of long prefill items when the grid is sparse
    int route = 0;               // 0 automatic, 1 tcgen05 route, 2 HBM route (everything on split-K)
    int num_sms = 148;
};
hg_status build_plan(const BatchView &v, int H_q, int H_kv, int d, const PlanOpts &o, Plan *p);

// O destinations of one attention call (AttnParams::outs).
struct OutSpec {
    int n = 0;
    uint16_t *ptr[kMaxOuts] = {};
    int64_t ld = 0;   // elements between token rows
    // entry barrier of a peer-window call, run by the fused step's append kernel
    // (world = 0: none; the caller launches its own barrier kernel)
    unsigned long long *bar_flags[kMaxOuts] = {};
    unsigned long long *bar_mine = nullptr;
    int bar_rank = 0, bar_world = 0;
    unsigned long long bar_epoch = 0;
    // set by the call when its append ran on a side stream without a stream join
    // (sharded HBM route): the caller's exit barrier waits for *wait_cnt >= wait_target
    mutable const unsigned long long *wait_cnt = nullptr;
    mutable unsigned long long wait_target = 0;
    // exit barrier epoch the call may fold into its last kernel (0: the caller launches
    // the exit barrier); the call sets exit_folded when it did
    unsigned long long exit_epoch = 0;
    mutable bool exit_folded = false;
};
hg_status attention_to(hg_kv_pool *pool, const hg_batch *batch, int32_t H_q, const void *q, const OutSpec &outs,
                       void *ws, size_t ws_bytes, void *stream);
hg_status plan_attention(hg_kv_pool *pool, const hg_batch *batch, int32_t H_q, bool append, size_t *bytes,
                         const hg_attn_opts *o = nullptr);
hg_status attention_planned(hg_kv_pool *pool, const hg_batch *batch, int32_t H_q, const void *q,
                            const void *k_new, const void *v_new, void *out, const OutSpec *outs, void *ws,
                            size_t ws_bytes, void *stream, const hg_attn_opts *o = nullptr);

// ---- kernel launchers (kernels.cu / tc_attn.cu) -----------------------------
hg_status launch_append(const uint16_t *k_new, const uint16_t *v_new, uint16_t *k_cache,
                        uint16_t *v_cache, const int64_t *slot, int T, int H_kv, int d,
                        void *stream);
// wave >= 0: only tokens whose TokDev.wave == wave (the pipelined host step
// appends the decode rows' K/V as soon as their wave of inputs has landed).
hg_status launch_append_dev(const AttnParams &p, const uint16_t *k_new, const uint16_t *v_new, int T, void *stream,
                            int wave = -1);
// Fused-step append with the slots in the kernel parameters (T <= kParamSlots):
// independent of the descriptor upload.
constexpr int kParamSlots = 3968;   // 31 KB of int64 slots (kernel parameter limit 32764 B)
// bar: AttnParams whose bar_* fields carry a peer-window entry barrier (NULL / bar_world = 0: none)
hg_status launch_append_param(const uint16_t *k_new, const uint16_t *v_new, uint16_t *k_cache, uint16_t *v_cache,
                              const int64_t *slots_host, int T, int H_kv, int d, void *stream,
                              const AttnParams *bar = nullptr);
// RoPE in the append prologue (NEXT-4): K rotated at its position before it is
// written, V copied, and (q_dst != NULL) Q rotated into q_dst.  Token slots and
// positions from the attention descriptors (fused step) or from arrays.
struct RopeArgs {
    double theta = 0;
    int rot = 0;   // rotary dims R (multiple of 16); 0 = none
};
hg_status launch_rope_append_dev(const AttnParams &p, const uint16_t *k_new, const uint16_t *v_new,
                                 const uint16_t *q_src, uint16_t *q_dst, int T, const RopeArgs &r, void *stream);
hg_status launch_rope_append(const uint16_t *k_new, const uint16_t *v_new, uint16_t *k_cache, uint16_t *v_cache,
                             const int64_t *slot, const int32_t *pos, int T, int H_kv, int d, const RopeArgs &r,
                             void *stream);
hg_status launch_splitk(const AttnParams &p, void *stream);
hg_status launch_peer_barrier(unsigned long long *const *flags, unsigned long long *mine, int rank, int world,
                              unsigned long long epoch, void *stream, bool pdl = false,
                              const unsigned long long *wait_cnt = nullptr, unsigned long long wait_target = 0);
// pdl: launched as a programmatic dependent of the kernel before it in `stream`
hg_status launch_combine(const AttnParams &p, void *stream, bool pdl = false);
hg_status launch_tc(const AttnParams &p, const void *tmap_k, const void *tmap_v, void *stream);
int tc_supported(int d);

}  // namespace hg
