/*
 * hygen.h -- C ABI of the B200-native hybrid-batch attention library
 * (HyGen, arXiv 2501.14808: one serving iteration's attention over a paged KV
 * cache, with the batch-latency predictor that prices it).
 *
 * Citations: P:n = /root/reference/PAPER.md line n (LaTeX source of the paper),
 * S:n = SPEC.md line n, "§8(x)" = SURVEY.md section.
 *
 * Conventions for every entry point
 *   - Returns hg_status (HG_OK = 0) unless stated; on error a thread-local
 *     message is available from hg_last_error() and NOTHING has been written
 *     (no device buffer, no pool metadata): validation precedes any launch.
 *   - Device pointers are CUDA device addresses on the pool's device; host
 *     pointers are ordinary (pageable or pinned) memory.  The caller owns all
 *     device buffers (KV cache, q, out, lse, workspace) and all streams.
 *   - `stream` is a cudaStream_t passed as void*; kernels are enqueued on it
 *     and the call returns without synchronising.  A CUDA error raised by an
 *     earlier launch surfaces as HG_E_CUDA on the next call.
 *   - Element types: bf16 = IEEE bfloat16 stored as uint16; fp32; int32.
 *   - Thread safety: one pool per thread at a time (no internal locking).
 */
#ifndef HYGEN_H_
#define HYGEN_H_

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define HG_API __attribute__((visibility("default")))
#else
#define HG_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    HG_OK = 0,
    HG_E_INVALID = 1,        /* contract violation in arguments or batch */
    HG_E_OOM = 2,            /* allocator cannot satisfy the request; message names the free count */
    HG_E_SHARED_WRITE = 3,   /* append would write into a shared (read-only) prefix block */
    HG_E_RANK_DEFICIENT = 4, /* predictor design matrix is rank deficient */
    HG_E_CUDA = 5,           /* a CUDA runtime / driver call failed */
    HG_E_NCCL = 6,           /* an NCCL call failed or NCCL is unavailable */
    HG_E_UNSUPPORTED = 7     /* valid request outside what this build implements (e.g. head_dim) */
} hg_status;

/* Message for the last non-OK status returned on this thread ("" if none). */
HG_API const char *hg_last_error(void);

/* GET_NUM_BLOCKS(l) of Alg. 1: ceil(tokens / block_size),
 * 0 for tokens <= 0.  Returns -1 if block_size < 1. */
HG_API int32_t hg_get_num_blocks(int32_t tokens, int32_t block_size);

/* ------------------------------------------------------------------------ */
/* KV block pool (memory budget m of Alg. 1)        */
/* ------------------------------------------------------------------------ */
typedef struct hg_kv_pool hg_kv_pool; /* opaque: allocator metadata + TMA descriptors */

typedef struct {
    int32_t num_blocks;   /* N_blk >= 1 */
    int32_t block_size;   /* B tokens per block: 16 (every shipped config; the only size this build accepts) */
    int32_t num_kv_heads; /* KV heads held by THIS rank (H_kv / G under head sharding) */
    int32_t head_dim;     /* d: 64 or 128 */
    int32_t device;       /* CUDA ordinal of k_cache / v_cache */
    void *k_cache;        /* caller-owned device bf16 [num_blocks][num_kv_heads][block_size][head_dim] */
    void *v_cache;        /* same layout; 16-byte aligned */
} hg_kv_pool_desc;

HG_API hg_status hg_kv_pool_create(const hg_kv_pool_desc *desc, hg_kv_pool **out);
HG_API hg_status hg_kv_pool_destroy(hg_kv_pool *pool);

/* All-or-nothing allocation of n blocks: the n smallest free ids in ascending
 * order, each with refcount 1 (deterministic, so head-sharded ranks make the
 * same decisions with no metadata traffic, §8(e)).  HG_E_OOM if fewer than n
 * are free (message: "need n, free f"). */
HG_API hg_status hg_kv_alloc(hg_kv_pool *pool, int32_t n, int32_t *out_ids);
/* refcount += 1 for each id (PSM prefix sharing).  All ids must be
 * allocated, else HG_E_INVALID and nothing changes. */
HG_API hg_status hg_kv_retain(hg_kv_pool *pool, const int32_t *ids, int32_t n);
/* refcount -= 1 for each id (repeats count), freeing at 0.  HG_E_INVALID if
 * any id would go below 0; nothing changes then. */
HG_API hg_status hg_kv_release(hg_kv_pool *pool, const int32_t *ids, int32_t n);
HG_API int32_t hg_kv_num_free(const hg_kv_pool *pool);
HG_API int32_t hg_kv_refcount(const hg_kv_pool *pool, int32_t id); /* -1 if id out of range */

/* ------------------------------------------------------------------------ */
/* The batch: B = {(r, l, t_req)} of Alg. 1, extended with the  */
/* paged-cache state of each request.                                        */
/* ------------------------------------------------------------------------ */
typedef struct {
    int32_t num_reqs;            /* R >= 0 */
    int32_t max_blocks_per_req;  /* W: row stride of block_table */
    const int32_t *block_table;  /* host [R][W]; entries past GET_NUM_BLOCKS(c_i+n_i) ignored (-1 by convention) */
    const int32_t *cached_len;   /* host [R]: c_i >= 0, tokens already in the cache */
    const int32_t *new_len;      /* host [R]: n_i >= 1 new tokens this iteration (l of Alg. 1; 1 = decode) */
    const uint8_t *is_offline;   /* host [R] or NULL: 0 online / 1 offline; no numeric effect (reading R6) */
    const int32_t *shared_prefix_blocks; /* host [R] or NULL: s_i, block_table[i][0:s_i] are shared read-only
                                            prefix blocks (PSM).  The shared sequences must form
                                            a trie (nested prefixes, e.g. system prompt -> few-shot block):
                                            an id listed by several rows sits at the same column in each,
                                            after identical ids; an id in one row's shared prefix appears
                                            in no other row's private part (else HG_E_INVALID) */
} hg_batch;

/* Write the new tokens' K and V rows into the cache: token j of request i
 * (batch row t = cu_q[i] + j) goes to position p = c_i + j, i.e. block
 * block_table[i][p / B], offset p % B, for every KV head.  k_new / v_new:
 * device bf16 [T][H_kv][d], T = sum n_i.  Bit-exact copy.  HG_E_SHARED_WRITE
 * if some p < s_i * B. */
HG_API hg_status hg_kv_append(hg_kv_pool *pool, const hg_batch *batch, const void *k_new,
                       const void *v_new, void *stream);

/* Rotary position embedding applied in the append / step prologue (SURVEY
 * §8(f) NEXT-4 "fuse append + RoPE into the prologue"; the paper's models are
 * Llama-family).  Rotate-half convention (Llama): with R = rotary_dim
 * and f_i = theta^(-2i/R), a row x at absolute position p becomes, for i < R/2,
 *   y[i]       = x[i] cos(p f_i) - x[i + R/2] sin(p f_i)
 *   y[i + R/2] = x[i + R/2] cos(p f_i) + x[i] sin(p f_i)
 * and y[i] = x[i] for i >= R.  Angles in fp64, rotation in fp32, result rounded
 * to bf16 (the cache dtype; reading R24). */
typedef struct {
    double theta;         /* base: 1e4 (Llama-2), 5e5 (Llama-3) */
    int32_t rotary_dim;   /* R: multiple of 16, <= head_dim; 0 = head_dim */
} hg_rope;

/* hg_kv_append with K rotated at its position p = c_i + j before it is
 * written (V copied).  Same validation; HG_E_INVALID for a bad rope. */
HG_API hg_status hg_kv_append_rope(hg_kv_pool *pool, const hg_batch *batch, const void *k_new,
                            const void *v_new, const hg_rope *rope, void *stream);

/* Tuning / test switches for hg_hybrid_attention_ex (zero-initialise for defaults). */
typedef struct {
    int32_t split_tokens;       /* >0: fixed split-K chunk (multiple of B) for decode rows, making the
                                   plan independent of load (bitwise reproducible across G, reading R18;
                                   prefill key cuts are off in this mode);
                                   0: automatic (sized to fill the SMs) */
    int32_t disable_prefix_pass;/* 1: no shared-prefix group pass (shared blocks read per request) */
    int32_t disable_tc;         /* 1: no tcgen05 kernel at all (prefill rows on split-K; shared prefixes
                                   as stacked-row split-K items when G_q <= 16) */
    int32_t num_sms;            /* 0: device SM count */
    void *events[6];            /* profiling: cudaEvent_t (or NULL) recorded on the stream right before /
                                   after the tcgen05 kernel [0,1], the split-K kernel [2,3] and the
                                   combine kernel [4,5] (bench.py's per-kernel roofline timing); when
                                   split-K merges the partials itself, [4,5] are both recorded where the
                                   combine would run (after every attention kernel) */
    void *debug_trace;          /* NULL, or device int64[4096]: clock64 stamps of tcgen05 CTA 0's pipeline
                                   events (kernel development aid; see tc_attn.cu) */
    const hg_rope *rope;        /* hg_hybrid_step only (NULL: none): q and k_new are pre-rotary; the
                                   append prologue rotates k_new into the cache and q into a workspace
                                   copy that the attention kernels read (cached keys were appended with
                                   the same rope).  HG_E_INVALID in hg_hybrid_attention_ex. */
    int32_t disable_prefill_split; /* 1: never cut a prefill chunk's keys into ranges.  0 (default): when
                                   the prefill items would fill < half the SMs, each chunk's cached keys
                                   are cut at KV-tile boundaries into ranges written as partials and
                                   merged by the combine kernel (small chunks at long contexts) */
    void *debug_sk_trace;       /* NULL, or device int64[2 * CTAs of the split-K grid]: %globaltimer (ns) at
                                   each split-K CTA's start and end, CTA (x, g) at 2 * (g * grid.x + x)
                                   (kernel development aid: the grid's occupancy over time) */
    int32_t route;              /* 0 (default): automatic -- the HBM route when the prefill work is small
                                   next to the decode pass, else the tcgen05 route; 1: tcgen05 route
                                   (prefill chunks and shared-prefix nodes on tcgen05 tiles); 2: HBM
                                   route (everything on the split-K kernel, prefix nodes as stacked-row
                                   split-K items; same as disable_tc for the prefill rows); 3: prefill
                                   chunks on tcgen05 tiles, shared-prefix nodes as stacked-row split-K
                                   items (G_q <= 16; above, on tiles as in route 1) -- no tile writes
                                   partials, so split-K merges every partial itself (the host step's
                                   route for mixed batches) */
} hg_attn_opts;

/* Bytes of device workspace hg_hybrid_attention needs for this batch. */
HG_API hg_status hg_hybrid_attention_workspace_size(const hg_kv_pool *pool, const hg_batch *batch,
                                             int32_t num_q_heads, size_t *bytes);

/* One hybrid iteration's attention.  For request i,
 * row j, q-head h (KV head g = h / (H_q/H_kv), reading R4):
 *   O[t][h] = softmax_p( q . K_i(p) / sqrt(d) ) . V_i(p),  p = 0 .. c_i + j
 * (causal, aligned to absolute positions -- chunked prefill P:63; decode
 * rows n_i = 1 see c_i + 1 keys; quadratic/linear cost of P:188).
 *   q   device bf16 [T][H_q][d], rows in request order
 *   out device bf16 [T][H_q][d]
 *   lse device fp32 [T][H_q] (natural log-sum-exp of the scaled scores) or NULL
 * The new tokens' K/V must already be in the cache (hg_kv_append earlier on
 * the same stream).  Descriptors are staged through pinned host memory and
 * copied into `workspace` on `stream`. */
HG_API hg_status hg_hybrid_attention(hg_kv_pool *pool, const hg_batch *batch, int32_t num_q_heads,
                              const void *q, void *out, float *lse, void *workspace,
                              size_t workspace_bytes, void *stream);
HG_API hg_status hg_hybrid_attention_ex(hg_kv_pool *pool, const hg_batch *batch, int32_t num_q_heads,
                                 const void *q, void *out, float *lse, void *workspace,
                                 size_t workspace_bytes, void *stream, const hg_attn_opts *opts);

/* Fused serving step on DEVICE buffers: hg_kv_append followed by
 * hg_hybrid_attention_ex with one validation (append rules included), one plan
 * and one descriptor upload; the append kernel derives each token's slot on the
 * device from the attention descriptors.  Arguments as in the two calls;
 * workspace from hg_hybrid_attention_workspace_size; opts may be NULL. */
HG_API hg_status hg_hybrid_step(hg_kv_pool *pool, const hg_batch *batch, int32_t num_q_heads, const void *q,
                                const void *k_new, const void *v_new, void *out, float *lse, void *workspace,
                                size_t workspace_bytes, void *stream, const hg_attn_opts *opts);

/* End-to-end serving step with HOST buffers (the e2e measurement of the
 * bench): q/k_new/v_new (host bf16 [T][H][d], pinned for async overlap) are
 * copied into the workspace, appended and attended, and out_host [T][H_q][d]
 * receives O.  Pipelined in two input waves on library-owned streams (a copy
 * stream and a high-priority tcgen05 stream, ordered after the caller's
 * `stream`): the decode rows' (n_i = 1) Q/K/V go up first and feed their
 * append + split-K on `stream` while the prefill-chunk rows' copies are still in
 * flight; those feed their append + the tcgen05 tiles, whose O rows are copied
 * back as soon as the tiles end; the decode rows' O follows the combine.
 * (One wave -- all copies, then the fused step -- when a decode item would read
 * a prefill row, e.g. head_dim without tcgen05 support, or with RoPE.)  Same
 * validation and errors as hg_hybrid_step; nothing is copied or launched on
 * error.  Synchronises `stream` (which has joined the library streams) before
 * returning, so out_host is valid and the host buffers may be reused.
 * Workspace: hg_hybrid_step_host_workspace_size (device copies of q, out,
 * k_new, v_new first, then the attention workspace).  The decode rows' copies
 * are queued before validation; on an error they are drained before the call
 * returns and nothing else is launched. */
HG_API hg_status hg_hybrid_step_host(hg_kv_pool *pool, const hg_batch *batch, int32_t num_q_heads,
                              const void *q_host, const void *k_new_host, const void *v_new_host,
                              void *out_host, void *workspace, size_t workspace_bytes, void *stream);
/* Pipelined use of the host step (a serving loop planning the next batch while the
 * GPU runs the current one):
 *   hg_hybrid_step_host_plan validates and plans `batch` for the NEXT host step into a
 *   second plan slot of the pool (pure host work; same errors as the step's
 *   validation; overwrites any earlier plan-ahead).
 *   hg_hybrid_step_host_async is hg_hybrid_step_host without the final synchronise:
 *   it returns once everything is queued on `stream`; out_host is valid, and the
 *   host input buffers may be reused, only after `stream` completes.  When the
 *   pool holds a plan-ahead for this same `batch` pointer, num_q_heads, shape and
 *   per-request lengths it is used instead of planning again -- the caller must not
 *   change the block-table contents in between (only their address is compared).
 *   Either way the plan-ahead is consumed.
 * A loop: plan(b0); for k: async(b_k); plan(b_{k+1}); synchronise(stream); ... keeps
 * each step's input upload after the previous step's result (the data dependency of
 * autoregressive decoding) and takes the validation and planning off the GPU's
 * critical path. */
HG_API hg_status hg_hybrid_step_host_plan(hg_kv_pool *pool, const hg_batch *batch, int32_t num_q_heads);
HG_API hg_status hg_hybrid_step_host_async(hg_kv_pool *pool, const hg_batch *batch, int32_t num_q_heads,
                                           const void *q_host, const void *k_new_host, const void *v_new_host,
                                           void *out_host, void *workspace, size_t workspace_bytes, void *stream);
HG_API hg_status hg_hybrid_step_host_workspace_size(const hg_kv_pool *pool, const hg_batch *batch,
                                             int32_t num_q_heads, size_t *bytes);

/* Derived integer outputs, host arrays:
 *   cu_q [R+1], kv_len [R], slot [T] = block_table[i][p/B]*B + p%B,
 *   prefix_group [R]: -1 if s_i = 0, else groups numbered by first appearance. */
HG_API hg_status hg_batch_indices(const hg_kv_pool *pool, const hg_batch *batch, int32_t *cu_q,
                           int32_t *kv_len, int64_t *slot, int32_t *prefix_group);

/* Plan statistics of the last attention call on this pool (for tests/bench). */
typedef struct {
    int32_t tc_tiles;        /* tcgen05 tiles (prefill + prefix group) */
    int32_t prefix_tiles;    /* of which shared-prefix group tiles */
    int32_t splitk_items;    /* split-K work items */
    int32_t combine_rows;    /* (token, KV head) pairs merged by the combine kernel */
    int32_t kernels;         /* kernels launched by the call */
    int64_t kv_bytes_unique; /* algorithmic KV bytes: 4*d*H_kv*U */
    int64_t kv_bytes_read;   /* KV bytes the plan streams from HBM */
    int32_t append_mode;     /* fused step's append: 0 its own kernel (or none), 1 inside the
                                tcgen05 kernel before its pipelines, 2 on the tcgen05 CTAs'
                                idle warp in the background (hidden behind cached-prefix tiles) */
} hg_plan_stats;
HG_API hg_status hg_last_plan_stats(const hg_kv_pool *pool, hg_plan_stats *out);

/* Host-only plan inspection (tests, no GPU): validates `batch` against a pool
 * of num_blocks blocks and builds the work plan hg_hybrid_attention would run
 * (use_tc = 1: as on a device with the tcgen05 path; num_sms: the grid it is
 * sized for), then lists, for every query row (token t, q head h) of every work
 * item, the key range [k0, k1) it attends there (causal cap applied) and the
 * partial index it writes (-1: the row's only range, written directly).
 * kind: 0 prefill tile (tcgen05), 1 shared-prefix node tile (tcgen05), 2
 * split-K item, 3 shared-prefix node as a stacked-row split-K item (HBM
 * route, see hg_attn_opts.route).  nparts: ranges the token's rows are merged from.  The ranges of
 * a row must tile [0, c_i + j + 1) exactly once -- the a.4 tile map, the split-K
 * plan and the prefill key cuts are checked that way.  Writes min(cap, total)
 * rows; *n_rows = total. */
typedef struct {
    int32_t t, h, k0, k1, part, kind, nparts;
} hg_plan_row;
HG_API hg_status hg_plan_rows(const hg_batch *batch, int32_t num_q_heads, int32_t num_kv_heads, int32_t head_dim,
                              int32_t num_blocks, int32_t num_sms, int32_t use_tc, const hg_attn_opts *opts,
                              hg_plan_row *rows, int64_t cap, int64_t *n_rows);

/* ------------------------------------------------------------------------ */
/* Multi-GPU: KV-head sharding + all-gather of outputs (§8(e); TP)    */
/* ------------------------------------------------------------------------ */
typedef struct hg_comm hg_comm;
/* Writes a 128-byte NCCL unique id (rank 0 creates it; broadcast it with
 * torch.distributed).  HG_E_NCCL if libnccl.so.2 cannot be loaded. */
HG_API hg_status hg_comm_unique_id(void *out_128_bytes);
/* nccl_unique_id NULL: a communicator without NCCL, usable only through a
 * peer window (below).  world <= 8. */
HG_API hg_status hg_comm_init(const void *nccl_unique_id, int32_t rank, int32_t world, int32_t device,
                       hg_comm **out);
HG_API hg_status hg_comm_destroy(hg_comm *comm);
/* Peer window (SURVEY §8(e) "v2 fuses the gather"): a library-owned device
 * buffer of `bytes` on every rank, mapped into every other rank with CUDA IPC
 * (NVLink peer memory).  Once open, hg_hybrid_attention_tp makes every
 * attention epilogue store its O rows straight into all ranks' windows at this
 * rank's head offset of [T][H_q][d] -- the all-gather is done by the kernels,
 * with no NCCL call and no transpose -- bracketed by two system-scope flag
 * barriers (entry: no rank overwrites a window its owner may still be reading;
 * exit: every rank's rows have landed).  The gathered O is then at *window_out;
 * it is copied to out_gathered unless out_gathered == *window_out.  A rank that
 * never reaches a barrier makes the others trap after ~30 s (HG_E_CUDA).
 * Steps, collectively on every rank:
 *   hg_comm_window_create(comm, bytes, handle, &win)  -> HG_IPC_HANDLE_BYTES opaque bytes
 *   all-gather the handles (e.g. torch.distributed), rank-major [world][64]
 *   hg_comm_window_open(comm, handles)
 * Calls whose T*H_q*d*2 exceeds `bytes` fall back to the NCCL path (HG_E_INVALID
 * if the communicator has none).  Readers of the window must be ordered before
 * the next hg_hybrid_attention_tp on the same stream. */
/* TP-native attention epilogue: the output projection of
 * the sharded attention fused with its reduce-scatter.  Rank r holds
 * O_r [T][K] (its heads' attention output, K = H_q/G * d) and the matching rows
 * of the projection W_r [K][N] (row-major, N = hidden); the layer output is
 * Y = sum_r O_r W_r [T][N], reduce-scattered by tokens: rank o receives rows
 * [o T/G, (o+1) T/G) into y_shard.  One tcgen05 GEMM kernel computes O_r W_r
 * and its epilogue stores each finished row (bf16) into the owning rank's
 * receive slot [r] of the peer window (so the transfer overlaps the GEMM),
 * then after a flag barrier each rank sums its G slots in fp32 (reading R25:
 * partials are rounded to bf16 once, as a bf16 reduce-scatter would carry
 * them).  G = 1: y_shard = O W directly.  Needs K % 64 == 0 and N % 128 == 0
 * (HG_E_UNSUPPORTED) and, for G > 1, an open window of G*ceil(T/G)*N*2 bytes. */
HG_API hg_status hg_out_proj_rs(hg_comm *comm, int32_t T, int32_t K, int32_t N, const void *o_local,
                         const void *w_local, void *y_shard, void *stream);
/* hg_hybrid_attention on this rank's heads (O kept in the workspace) followed by
 * hg_out_proj_rs: the sharded attention layer without an output all-gather. */
HG_API hg_status hg_hybrid_attention_tp_proj_workspace_size(const hg_kv_pool *pool, const hg_comm *comm,
                                                     const hg_batch *batch, int32_t num_q_heads_total,
                                                     size_t *bytes);
HG_API hg_status hg_hybrid_attention_tp_proj(hg_kv_pool *pool, hg_comm *comm, const hg_batch *batch,
                                      int32_t num_q_heads_total, const void *q_local, const void *w_local,
                                      int32_t N, void *y_shard, void *workspace, size_t workspace_bytes,
                                      void *stream);

#define HG_IPC_HANDLE_BYTES 64
HG_API hg_status hg_comm_window_create(hg_comm *comm, size_t bytes, void *ipc_handle_out, void **window_out);
HG_API hg_status hg_comm_window_open(hg_comm *comm, const void *handles);
/* Rank r holds KV heads [r*H_kv/G, (r+1)*H_kv/G) in `pool` and q-heads
 * [r*H_q/G, (r+1)*H_q/G) in q_local ([T][H_q/G][d]); every rank receives the
 * full out_gathered [T][H_q][d].  workspace must hold
 * hg_hybrid_attention_tp_workspace_size bytes. */
HG_API hg_status hg_hybrid_attention_tp_workspace_size(const hg_kv_pool *pool, const hg_comm *comm,
                                                const hg_batch *batch, int32_t num_q_heads_total,
                                                size_t *bytes);
HG_API hg_status hg_hybrid_attention_tp(hg_kv_pool *pool, hg_comm *comm, const hg_batch *batch,
                                 int32_t num_q_heads_total, const void *q_local, void *out_gathered,
                                 void *workspace, size_t workspace_bytes, void *stream);
/* The sharded serving step: hg_kv_append of this rank's KV-head slice
 * (k_new_local / v_new_local, dev bf16 [T][H_kv_local][d]) fused with
 * hg_hybrid_attention_tp, as hg_hybrid_step fuses them on one GPU (one
 * validation with the append rules, one plan, one descriptor upload, the slots
 * derived on the device).  Same workspace, window and error rules as
 * hg_hybrid_attention_tp. */
/* hg_hybrid_attention_tp with plan options (hg_attn_opts, nullable; events and
 * the rope prologue do not apply).  With opts->split_tokens > 0 the plan is
 * load-independent (reading R17): every rank's slice, and so the gathered O, is
 * bit-identical to the unsharded call with the same split, whatever G. */
HG_API hg_status hg_hybrid_attention_tp_ex(hg_kv_pool *pool, hg_comm *comm, const hg_batch *batch,
                                           int32_t num_q_heads_total, const void *q_local, void *out_gathered,
                                           void *workspace, size_t workspace_bytes, void *stream,
                                           const hg_attn_opts *opts);
HG_API hg_status hg_hybrid_step_tp(hg_kv_pool *pool, hg_comm *comm, const hg_batch *batch,
                                   int32_t num_q_heads_total, const void *q_local, const void *k_new_local,
                                   const void *v_new_local, void *out_gathered, void *workspace,
                                   size_t workspace_bytes, void *stream);
/* hg_hybrid_step_tp with plan options (nullable; per-kernel events recorded as
 * in hg_hybrid_attention_ex, no rope: HG_E_INVALID). */
HG_API hg_status hg_hybrid_step_tp_ex(hg_kv_pool *pool, hg_comm *comm, const hg_batch *batch,
                                      int32_t num_q_heads_total, const void *q_local, const void *k_new_local,
                                      const void *v_new_local, void *out_gathered, void *workspace,
                                      size_t workspace_bytes, void *stream, const hg_attn_opts *opts);

/* ------------------------------------------------------------------------ */
/* Batch-latency predictor (§4.2 Eq. 1; App. B Eq. 2)  */
/* ------------------------------------------------------------------------ */
/* Feature k has weight w[1+k]; w[0] is the intercept. */
typedef struct {
    double S_p;   /* 0: total prefill tokens */
    double S_d;   /* 1: total decode tokens (= N_d: one token per decode) */
    double S_p2;  /* 2: S_p^2 (Eq. 1) */
    double S_d2;  /* 3: S_d^2 (Eq. 1 only) */
    double N_p;   /* 4: prefill requests */
    double N_d;   /* 5: decode requests */
    double P2;    /* 6: attended prefill pairs sum n_i (c_i + (n_i+1)/2) (reading R14) */
    double D_ctx; /* 7: unique KV tokens read by decode rows (reading R15) */
} hg_features;

#define HG_FEAT_S_P   (1 << 0)
#define HG_FEAT_S_D   (1 << 1)
#define HG_FEAT_S_P2  (1 << 2)
#define HG_FEAT_S_D2  (1 << 3)
#define HG_FEAT_N_P   (1 << 4)
#define HG_FEAT_N_D   (1 << 5)
#define HG_FEAT_P2    (1 << 6)
#define HG_FEAT_D_CTX (1 << 7)
/* Eq. 1 with the collinear S_d (= N_d) dropped, and the attention-aware fit. */
#define HG_MASK_EQ1   (HG_FEAT_S_P | HG_FEAT_S_P2 | HG_FEAT_S_D2 | HG_FEAT_N_P | HG_FEAT_N_D)
#define HG_MASK_EQ2   (HG_FEAT_S_P | HG_FEAT_S_P2 | HG_FEAT_N_P | HG_FEAT_N_D)
#define HG_MASK_ATTN  (HG_FEAT_S_P | HG_FEAT_P2 | HG_FEAT_D_CTX | HG_FEAT_N_D | HG_FEAT_N_P)
/* Fit option (OR into the mask): minimise the squared RELATIVE error
 * sum_i ((w.x_i - y_i) / y_i)^2 -- linear regression weighted by 1 / y_i^2, the
 * least-squares criterion closest to the MAPE the paper reports;
 * requires every y_i > 0. */
#define HG_FIT_RELATIVE (1 << 8)

typedef struct {
    double w[9];          /* w[0] intercept, w[1+k] feature k (0 for unselected) */
    int32_t feature_mask; /* HG_FEAT_* bits used by the fit (| HG_FIT_RELATIVE if set) */
    int32_t n_samples;
    double train_mape;    /* mean |pred - y| / y on the training set */
} hg_predictor;

/* Features of a batch (decode row iff n_i == 1 and c_i >= 1, reading R5;
 * shared prefixes counted once per group in D_ctx). */
HG_API hg_status hg_batch_features(const hg_batch *batch, int32_t block_size, hg_features *out);
/* Ordinary least squares of y_ms on [1, selected features] ("linear
 * regression"), Householder QR in fp64 on column-scaled data.
 * HG_E_RANK_DEFICIENT if the design has rank < 1 + popcount(mask). */
HG_API hg_status hg_predictor_fit(const hg_features *X, const double *y_ms, int32_t n, int32_t feature_mask,
                           hg_predictor *out);
/* w . [1, x], floored at 0. */
HG_API double hg_predictor_predict(const hg_predictor *model, const hg_features *x);

/* ------------------------------------------------------------------------ */
/* SLO-aware batch composition (Alg. 1 SLO_AWARE_SCHEDULE)       */
/* ------------------------------------------------------------------------ */
typedef struct {
    int32_t cached;               /* tokens already in the KV cache */
    int32_t prompt_left;          /* prompt tokens not yet prefilled; 0 => the request decodes */
    int32_t shared_prefix_tokens; /* tokens of a physically shared prefix (D_ctx counts it once per group) */
    int32_t group;                /* shared-prefix group, -1 if none */
} hg_sched_req;

typedef struct {
    int32_t index;  /* < n_running: running[index]; else queue[index - n_running] */
    int32_t tokens; /* l of Alg. 1: 0 for a decode step, else the prefill chunk */
    double t_req;   /* predicted marginal batch latency charged to the budget (ms) */
} hg_sched_entry;

/* The batch under construction across the phases of one iteration (Alg. 2
 * runs SLO_AWARE_SCHEDULE for the online, then the offline phase on ONE batch,
 * P:507-512).  Zero-initialise it once per iteration and pass it to every
 * phase together with the previous phase's *t_left / *c_left / *m_left: each
 * phase then prices its requests against the whole batch so far (the Eq. 1
 * cross terms such as 2 S_p l w_{S_p^2} included) and the intercept is charged
 * once.  NULL: the call is a batch of its own. */
#define HG_SCHED_MAX_GROUPS 256
typedef struct {
    double features[8];        /* hg_features order: features of the entries admitted so far */
    int32_t intercept_charged; /* 1 once w[0] has been taken off a budget */
    int32_t n_groups;          /* shared-prefix groups that already have a decode row */
    int32_t groups[HG_SCHED_MAX_GROUPS];
} hg_sched_state;

/* One scheduling pass (online or offline phase) of Alg. 1 with the fitted
 * predictor: running decodes first (admitted unconditionally when
 * phase_online, else only while t_req <= t), then prefilling running requests
 * and the queue in order, each given the largest chunk l that fits the
 * remaining latency t, chunk c and memory m budgets (get_max_tokens, P:156;
 * m decreases by GET_NUM_BLOCKS(l)); the first prefill that cannot be
 * given a token ends the pass (preemption is not modelled, reading R21).
 * t_req is the marginal increase of the batch prediction (clamped at 0); the
 * model intercept is charged once per batch (reading R19).  state (nullable,
 * in/out): the batch so far -- see hg_sched_state; HG_E_UNSUPPORTED if the
 * batch would hold more than HG_SCHED_MAX_GROUPS groups.  out must hold
 * n_running + n_queue entries; *t_left / *c_left / *m_left (nullable) return
 * the budgets left for the next phase (Alg. 2 runs the online then the
 * offline phase: pass them on with the same state). */
HG_API hg_status hg_slo_aware_schedule(const hg_predictor *model, int32_t block_size, const hg_sched_req *running,
                                       int32_t n_running, const hg_sched_req *queue, int32_t n_queue,
                                       double latency_budget_ms, int32_t chunk_budget, int32_t memory_blocks,
                                       int32_t phase_online, hg_sched_state *state, hg_sched_entry *out,
                                       int32_t *n_out, double *t_left, int32_t *c_left, int32_t *m_left);

/* ------------------------------------------------------------------------ */
/* Prefix Sharing Maximization (§4.3; Alg. 3)           */
/* ------------------------------------------------------------------------ */
typedef struct hg_psm hg_psm; /* prefix tree T_p over offline prompts */
HG_API hg_status hg_psm_create(hg_psm **out);
HG_API hg_status hg_psm_destroy(hg_psm *psm);
/* Insert request `request_id` (unique, >= 0) with its prompt tokens. */
HG_API hg_status hg_psm_insert(hg_psm *psm, int32_t request_id, const int32_t *tokens, int32_t n);
/* Remove a request (once scheduled).  HG_E_INVALID if absent. */
HG_API hg_status hg_psm_remove(hg_psm *psm, int32_t request_id);
HG_API int32_t hg_psm_size(const hg_psm *psm);
/* The first `max` requests in DFS order of the tree (a node's own requests in
 * insertion order, then its children in first-insertion order), and for each
 * the length of the prefix it shares with its DFS predecessor (0 for the first)
 * -- the shared-prefix length the attention kernel's prefix groups can reuse. */
HG_API hg_status hg_psm_dfs_order(hg_psm *psm, int32_t *ids, int32_t *lcp_with_prev, int32_t max, int32_t *n_out);
/* Alg. 3: running offline requests in order (a decode that does not fit the
 * remaining budget ends the pass -- the inverted gate of P:550 read as
 * `t < t_req => break`, reading R16; a prefill gets the largest fitting chunk or
 * ends the pass), then new requests in the tree's DFS order, each given the
 * largest fitting chunk (get_max_prefill) and removed from the tree.  by_id[k]
 * describes tree request k (n_ids entries).  out entries index running[] for
 * index < n_running, else request id + n_running.  Budgets, marginal
 * latencies and state (the online phase's batch) as in hg_slo_aware_schedule. */
HG_API hg_status hg_psm_offline_schedule(const hg_predictor *model, int32_t block_size, hg_psm *psm,
                                         const hg_sched_req *running, int32_t n_running, const hg_sched_req *by_id,
                                         int32_t n_ids, double latency_budget_ms, int32_t chunk_budget,
                                         int32_t memory_blocks, hg_sched_state *state, hg_sched_entry *out,
                                         int32_t *n_out, double *t_left, int32_t *c_left, int32_t *m_left);

#ifdef __cplusplus
}
#endif
#endif /* HYGEN_H_ */
