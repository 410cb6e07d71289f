// host.cpp -- host-side steps of the hot path:
// error reporting, batch validation (§8(b) rules), prefix groups, and the
// per-call work plan consumed by the sm_100a kernels.
#include <algorithm>
#include <climits>
#include <cstdlib>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <numeric>

#include "hg_internal.h"

namespace hg {

static thread_local char g_err[512] = "";

void set_error(const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof g_err, fmt, ap);
    va_end(ap);
}

hg_status fail(hg_status s, const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof g_err, fmt, ap);
    va_end(ap);
    return s;
}

static inline int ceil_div(int64_t a, int64_t b) { return (int)((a + b - 1) / b); }

hg_status view_batch(const hg_batch *b, BatchView *v) {
    if (!b) return fail(HG_E_INVALID, "batch is NULL");
    if (b->num_reqs < 0) return fail(HG_E_INVALID, "num_reqs < 0");
    v->R = b->num_reqs;
    v->W = b->max_blocks_per_req;
    v->bt = b->block_table;
    v->c = b->cached_len;
    v->n = b->new_len;
    if (v->R > 0 && (!v->bt || !v->c || !v->n || v->W < 1))
        return fail(HG_E_INVALID, "batch arrays missing or max_blocks_per_req < 1");
    if (b->shared_prefix_blocks) {
        v->s = b->shared_prefix_blocks;
    } else {
        v->s_store.assign((size_t)std::max(v->R, 1), 0);
        v->s = v->s_store.data();
    }
    return HG_OK;
}

// Per-thread scratch reused across calls: epoch-stamped per-block records for
// the shared (prefix) blocks of the batch (touched sum(s_i) times per call) and
// a bitmap over block ids (N_blk / 8 bytes, L1/L2 resident) for the duplicate /
// sharing rules.
struct Scratch {
    std::vector<uint64_t> stamp;  // epoch << 32 | column of the shared block
    std::vector<int32_t> par;     // id before it in every row that shares it (-1: column 0)
    std::vector<int32_t> gid;     // prefix group of the sequences ending at this block (-1: none yet)
    std::vector<int32_t> cnt;     // build_plan: prefix-pass rows whose shared path passes the block
    std::vector<int32_t> node;    // build_plan: tile-map node starting at the block (-1: none)
    uint32_t epoch = 0;
    std::vector<uint64_t> bm_priv;   // ids already used (shared prefixes, private blocks)
    std::vector<int32_t> group;   // prefix group of each row (valid after validate)
    std::vector<int32_t> owners;
    int64_t n_shared = 0;         // distinct shared block ids in the batch
    // build_plan: prefix-pass extent of each row and its tile-map nodes
    struct Node { int32_t a, e, rep, depth, nm, first; };
    std::vector<int32_t> pre_end, npre;
    std::vector<int32_t> np;      // key ranges of each prefill request (1: whole)
    std::vector<Node> nodes;
};
static thread_local Scratch g_scr;

static inline bool bm_test(const uint64_t *bm, uint32_t b) { return bm[b >> 6] >> (b & 63) & 1; }
static inline void bm_set(uint64_t *bm, uint32_t b) { bm[b >> 6] |= 1ull << (b & 63); }

hg_status validate(const BatchView &v, int B, int num_blocks, int num_q_heads, int H_kv, bool append) {
    if (num_q_heads >= 0) {
        if (H_kv <= 0 || num_q_heads <= 0 || num_q_heads % H_kv)
            return fail(HG_E_INVALID, "num_q_heads %d not a positive multiple of num_kv_heads %d",
                        num_q_heads, H_kv);
    }
    Scratch &sc = g_scr;
    const size_t words = ((size_t)num_blocks + 63) / 64;
    if (sc.stamp.size() < (size_t)num_blocks) {
        sc.stamp.assign((size_t)num_blocks, 0);
        sc.par.assign((size_t)num_blocks, -1);
        sc.gid.assign((size_t)num_blocks, -1);
        sc.cnt.assign((size_t)num_blocks, 0);
        sc.node.assign((size_t)num_blocks, -1);
    }
    if (sc.bm_priv.size() < words) sc.bm_priv.assign(words, 0);
    memset(sc.bm_priv.data(), 0, words * 8);
    if (++sc.epoch == 0) {
        std::fill(sc.stamp.begin(), sc.stamp.end(), 0);
        sc.epoch = 1;
    }
    const uint64_t ep = (uint64_t)sc.epoch << 32;
    sc.group.assign((size_t)v.R, -1);
    sc.owners.clear();
    int ng = 0, shared_write = -1;
    sc.n_shared = 0;
    uint64_t *bp = sc.bm_priv.data();
    // One pass over the block table (it is read once: ~300 KB for a C3-sized batch):
    // shapes and id ranges; shared prefixes must form a trie (NEXT-3, R23):
    // a block shared by several rows sits at the same column in each, after the same
    // id (hence after identical sequences, by induction); every id is used by one
    // row's private columns or by shared prefixes, never both (bitmap of ids taken).
    for (int i = 0; i < v.R; ++i) {
        const int64_t c = v.c[i], n = v.n[i], s = v.s[i];
        if (n < 1 || c < 0 || s < 0)
            return fail(HG_E_INVALID, "request %d: need n>=1, c>=0, s>=0 (c=%lld n=%lld s=%lld)", i,
                        (long long)c, (long long)n, (long long)s);
        const int nb = ceil_div(c + n, B);
        if (nb > v.W) return fail(HG_E_INVALID, "request %d needs %d blocks > max_blocks_per_req %d", i, nb, v.W);
        if (s > nb) return fail(HG_E_INVALID, "request %d: shared blocks %lld > blocks %d", i, (long long)s, nb);
        if (append && c < s * B && shared_write < 0) shared_write = i;
        const int32_t *row = v.bt + (int64_t)i * v.W;
        for (int col = 0; col < s; ++col) {
            const int32_t b = row[col], parent = col ? row[col - 1] : -1;
            if ((uint32_t)b >= (uint32_t)num_blocks)
                return fail(HG_E_INVALID, "request %d: block id outside [0, %d)", i, num_blocks);
            const uint64_t t = sc.stamp[b];
            if ((t & ~0xFFFFFFFFull) == ep) {
                if ((int)(t & 0xFFFFFFFFu) != col || sc.par[b] != parent)
                    return fail(HG_E_INVALID, "request %d shares block %d but not an identical prefix before it",
                                i, b);
            } else {
                if (bm_test(bp, (uint32_t)b))
                    return fail(HG_E_INVALID, "block %d of request %d is also used by another row or prefix", b, i);
                sc.stamp[b] = ep | (uint32_t)col;
                sc.par[b] = parent;
                sc.gid[b] = -1;
                sc.cnt[b] = 0;
                sc.node[b] = -1;
                bm_set(bp, (uint32_t)b);
                ++sc.n_shared;
            }
        }
        // private columns: range check and test-and-set, branch-free per id
        uint32_t bad = 0;
        uint64_t seen = 0;
        for (int col = (int)s; col < nb; ++col) {
            const uint32_t b = (uint32_t)row[col];
            bad |= (uint32_t)(b >= (uint32_t)num_blocks);
            const uint32_t bb = b < (uint32_t)num_blocks ? b : 0u;
            uint64_t &w = bp[bb >> 6];
            const uint64_t bit = 1ull << (bb & 63);
            seen |= w & bit;
            w |= bit;
        }
        if (bad) return fail(HG_E_INVALID, "request %d: block id outside [0, %d)", i, num_blocks);
        if (seen) {
            for (int col = (int)s; col < nb; ++col)   // name the offending id (error path only)
                for (int k = (int)s; k < col; ++k)
                    if (row[k] == row[col])
                        return fail(HG_E_INVALID, "block %d of request %d is also used by another row or prefix",
                                    row[col], i);
            return fail(HG_E_INVALID, "a private block of request %d is also used by another row or prefix", i);
        }
        if (s > 0) {   // prefix group = identical whole shared sequence = same last shared block
            int32_t &g = sc.gid[row[s - 1]];
            if (g < 0) {
                g = ng++;
                sc.owners.push_back(i);
            }
            sc.group[i] = g;
        }
    }
    if (shared_write >= 0)
        return fail(HG_E_SHARED_WRITE, "request %d appends at position %d inside its shared prefix (%d blocks)",
                    shared_write, v.c[shared_write], v.s[shared_write]);
    return HG_OK;
}

void prefix_groups(const BatchView &v, std::vector<int32_t> *group) {
    // numbered by first appearance of the shared sequence (valid after validate())
    *group = g_scr.group;
    group->resize((size_t)v.R, -1);
}

static size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// LPT order (longest key range first) by counting sort on the range in blocks: O(n + range).
template <class Item>
static void lpt_sort(std::vector<Item> &v, std::vector<Item> &tmp) {
    if (v.size() < 2) return;
    int maxb = 0;
    for (const Item &it : v) maxb = std::max(maxb, (it.k1 - it.k0 + kBlock - 1) / kBlock);
    std::vector<int32_t> cnt((size_t)maxb + 2, 0);
    for (const Item &it : v) cnt[maxb - (it.k1 - it.k0 + kBlock - 1) / kBlock + 1]++;
    for (int k = 1; k <= maxb + 1; ++k) cnt[k] += cnt[k - 1];
    tmp.resize(v.size());
    for (const Item &it : v) tmp[cnt[maxb - (it.k1 - it.k0 + kBlock - 1) / kBlock]++] = it;
    v.swap(tmp);
}

// tcgen05 tiles: keep the tiles that read the same KV stream (same block table
// and KV head) adjacent, so the CTAs of one wave share K/V through L2, longest
// stream first and longest tile first within a stream (LPT at stream grain).
static void stream_sort(std::vector<TcItem> &v, std::vector<TcItem> &tmp) {
    const size_t n = v.size();
    if (n < 2) return;
    struct Seg { size_t b, e; int32_t len; };
    std::vector<Seg> segs;
    for (size_t a = 0; a < n;) {
        size_t b = a;
        int32_t mx = 0;
        while (b < n && v[b].bt_off == v[a].bt_off && v[b].g == v[a].g) {
            mx = std::max(mx, v[b].k1 - v[b].k0);
            ++b;
        }
        segs.push_back({a, b, mx});
        a = b;
    }
    std::stable_sort(segs.begin(), segs.end(), [](const Seg &x, const Seg &y) { return x.len > y.len; });
    tmp.clear();
    tmp.reserve(n);
    for (const Seg &s : segs) {
        const size_t first = tmp.size();
        tmp.insert(tmp.end(), v.begin() + s.b, v.begin() + s.e);
        std::stable_sort(tmp.begin() + first, tmp.end(),
                         [](const TcItem &x, const TcItem &y) { return (x.k1 - x.k0) > (y.k1 - y.k0); });
    }
    v.swap(tmp);
}

// Persistent tcgen05 grid: greedy LPT assignment of the items to the CTAs
// (longest first, each to the least-loaded CTA), so a CTA's items are a
// contiguous range.  Cost of an item = KV tiles x Q tiles (+1 for its Q load and
// epilogue).  A static round-robin of the sorted list instead gives CTA k items
// k, k + P, ...: on P1 (4 chunks at staggered offsets) its makespan is 1.4x the
// greedy one.
static void assign_tc(Plan *p) {
    const int P = p->tc_ctas, n = (int)p->tc.size();
    p->tc_off.assign((size_t)P + 1, 0);
    if (n == 0) return;
    auto cost = [](const TcItem &it) {
        return (int64_t)((it.k1 - it.k0 + kTcKeys - 1) / kTcKeys) * (it.nrows > kTcRows ? 2 : 1) + 1;
    };
    std::stable_sort(p->tc.begin(), p->tc.end(),
                     [&](const TcItem &a, const TcItem &b) { return cost(a) > cost(b); });
    using Slot = std::pair<int64_t, int32_t>;   // (load, cta): min-heap, ties to the lower CTA id
    std::vector<Slot> heap;
    heap.reserve((size_t)P);
    for (int b = 0; b < P; ++b) heap.push_back({0, b});
    std::vector<int32_t> owner((size_t)n);
    auto gt = [](const Slot &a, const Slot &b) { return a > b; };
    for (int k = 0; k < n; ++k) {
        std::pop_heap(heap.begin(), heap.end(), gt);
        owner[k] = heap.back().second;
        heap.back().first += cost(p->tc[k]);
        std::push_heap(heap.begin(), heap.end(), gt);
    }
    for (int k = 0; k < n; ++k) p->tc_off[owner[k] + 1]++;
    for (int b = 0; b < P; ++b) p->tc_off[b + 1] += p->tc_off[b];
    std::vector<int32_t> fill(p->tc_off.begin(), p->tc_off.end() - 1);
    p->tc_tmp.resize((size_t)n);
    for (int k = 0; k < n; ++k) p->tc_tmp[fill[owner[k]]++] = p->tc[k];
    p->tc.swap(p->tc_tmp);
}

hg_status build_plan(const BatchView &v, int H_q, int H_kv, int d, const PlanOpts &o, Plan *p) {
    const int G = H_q / H_kv;
    const int B = kBlock;
    p->R = v.R;
    p->W = v.W;
    p->reqs.resize((size_t)v.R);
    p->sk.clear();
    p->tc.clear();
    p->tc_tok.clear();
    p->comb.clear();
    p->n_slots = 0;
    p->prefix_tiles = 0;
    p->prefix_sk = 0;
    int64_t T = 0, nbt = 0;
    for (int i = 0; i < v.R; ++i) {
        p->reqs[i] = ReqDev{v.c[i], v.n[i], (int32_t)T, (int32_t)nbt, -1, 0, 0ull};
        T += v.n[i];
        nbt += ceil_div((int64_t)v.c[i] + v.n[i], B);
    }
    p->T = (int)T;
    p->n_bt = nbt;   // the block ids themselves go straight from the batch into the descriptor image
    p->tok.resize((size_t)T);
    for (int i = 0; i < v.R; ++i)
        for (int j = 0; j < v.n[i]; ++j) p->tok[(size_t)p->reqs[i].cu_q + j] = TokDev{-1, 1, i, 0};

    Scratch &sc = g_scr;
    const bool tc_ok = o.use_tc && tc_supported(d) && G <= kTcRows;
    // ---- a.4 tile map over the trie of shared prefixes (NEXT-3) -------------------
    // cnt[b] = decode rows whose shared path passes block b.  A row's prefix pass
    // covers its leading columns with cnt >= 2 (a lone member gains nothing; cnt
    // never grows along a path).  Those columns split into runs of equal cnt, i.e.
    // of one member set: each run is a node whose keys are read once for the
    // stacked rows of all its members, as partial `depth` of every member row.
    sc.pre_end.assign((size_t)v.R, 0);
    sc.npre.assign((size_t)v.R, 0);
    sc.nodes.clear();
    // A row takes part in a node only over whole blocks inside its causal range: a
    // node's tiles give every member the node's full key range (no per-row limit),
    // so a decode row whose context ends inside a shared block (plain
    // hg_hybrid_attention allows c_i + 1 < s_i * B) stops its pass at the last
    // block it sees completely, and split-K covers the rest.
    auto pass_cols = [&](int i) { return std::min<int64_t>(v.s[i], ((int64_t)v.c[i] + 1) / B); };
    if (o.prefix_pass && (tc_ok || G <= kSkRows)) {
        for (int i = 0; i < v.R; ++i)
            if (v.n[i] == 1 && v.s[i] > 0) {
                const int32_t *row = v.bt + (int64_t)i * v.W;
                for (int col = 0, e = (int)pass_cols(i); col < e; ++col) sc.cnt[row[col]]++;
            }
        for (int i = 0; i < v.R; ++i) {
            if (v.n[i] != 1 || v.s[i] == 0) continue;
            const int32_t *row = v.bt + (int64_t)i * v.W;
            const int cols = (int)pass_cols(i);
            int e = 0;
            while (e < cols && sc.cnt[row[e]] >= 2) ++e;
            sc.pre_end[i] = e;
            int a = 0, depth = 0;
            while (a < e) {
                const int32_t b = row[a];
                int z = a + 1;
                while (z < e && sc.cnt[row[z]] == sc.cnt[b]) ++z;
                if (sc.node[b] < 0) {
                    sc.node[b] = (int32_t)sc.nodes.size();
                    sc.nodes.push_back(Scratch::Node{a, z, i, depth, 0, 0});
                }
                sc.nodes[sc.node[b]].nm++;
                a = z;
                ++depth;
            }
            sc.npre[i] = depth;
        }
    }
    // ---- route: tcgen05 tiles for the prefill chunks and prefix nodes, or the
    // HBM route (everything on the split-K kernel, prefix nodes as stacked-row
    // split-K items).  Beside a decode pass the tcgen05 CTAs, which need whole
    // SMs, either wait for split-K's CTAs to drain or starve on TMA loads queued
    // behind its HBM traffic; when the prefill work is small next to the decode
    // pass, folding it into the HBM-bound kernel is cheaper (measured: c1 / c3
    // and their 8-way shards, tools/exp_shard.py), and split-K can then start
    // beside the append (it reads this call's new K/V from the step's inputs).
    bool tc_on = tc_ok && o.route != 2;
    if (tc_on && o.route == 0) {
        double dec_bytes = 0, pre_flops = 0;
        for (int i = 0; i < v.R; ++i) {
            if (v.n[i] == 1) dec_bytes += ((double)v.c[i] + 1 - (double)sc.pre_end[i] * B) * 4.0 * d * H_kv;
            else pre_flops += 4.0 * d * H_q * v.n[i] * ((double)v.c[i] + (v.n[i] + 1) / 2.0);
        }
        // prefill rows on mma.sync split-K items at ~300 TFLOP/s vs the decode pass at ~6.5 TB/s
        tc_on = !(dec_bytes > 0 && pre_flops / 300e12 < 0.5 * dec_bytes / 6.5e12);
    }
    // route 3: prefill chunks on tcgen05 tiles, shared-prefix nodes as stacked-row
    // split-K items (G_q <= 16) -- so no tcgen05 item writes partials and split-K
    // merges every partial itself (no combine kernel after it)
    const bool nodes_tc = tc_on && !(o.route == 3 && G <= kSkRows);
    if (!nodes_tc && !sc.nodes.empty()) {
        // HBM route: a node pays for its extra partials (every member row gets merged)
        // only when the members would re-read a large share of the KV bytes: a prefix
        // re-read by its members mostly hits L2.  Measured: c2_nested (re-reads 40 %
        // of its unique bytes) gains 1.5 % with the nodes, c2 (25 %) is even, c3
        // (12 %) loses 2 %.  No stacked-row split-K items above 16 rows (G_q > 16).
        double reread = 0, uniq = 0;
        for (int i = 0; i < v.R; ++i) uniq += (double)v.c[i] + v.n[i] - (double)v.s[i] * B;
        uniq += (double)sc.n_shared * B;
        for (const Scratch::Node &nd : sc.nodes) reread += (double)(nd.nm - 1) * (nd.e - nd.a) * B;
        if (G > kSkRows || ((o.route == 0 || o.route == 3) && reread <= 0.25 * uniq)) {
            std::fill(sc.pre_end.begin(), sc.pre_end.end(), 0);
            std::fill(sc.npre.begin(), sc.npre.end(), 0);
            sc.nodes.clear();
        }
    }
    // rows per tcgen05 CTA: 256 (two Q tiles sharing K/V, half the L2 traffic per
    // FLOP) when that still gives every SM a CTA, else 128 (more CTAs)
    int ipr = kTcRows;
    if (tc_on) {
        int64_t n256 = 0;
        for (int i = 0; i < v.R; ++i)
            if (v.n[i] > 1) n256 += (int64_t)H_kv * ceil_div((int64_t)v.n[i] * G, 2 * kTcRows);
        if (nodes_tc)
            for (const Scratch::Node &nd : sc.nodes) n256 += (int64_t)H_kv * ceil_div((int64_t)nd.nm * G, 2 * kTcRows);
        if (n256 >= o.num_sms) ipr = 2 * kTcRows;
        // Long prefill items on an unbalanced grid (a small chunk at a long prompt:
        // one item = one CTA walking thousands of keys while the other SMs run out
        // of work): cut such a request's keys into np_i ranges at KV-tile
        // boundaries inside its cached prefix (visible to every row), the last
        // range holding the causal diagonal; the ranges write partials that the
        // combine kernel merges like split-K's.  A 256-row item advances ~1.5 us
        // per 128-key tile and the decode rows' split-K pass is HBM-bound (~its
        // unique KV bytes / 6.5 TB/s): a chunk is cut only where its chain is
        // 1.5x longer than both that pass and the grid's average load, into pieces
        // no longer than the larger of the two (and >= 8 tiles).
        sc.np.assign((size_t)v.R, 1);
        constexpr double kTileUs = 1.5, kHbmBytesPerUs = 6.5e6;
        double dec_keys = 0;
        for (int i = 0; i < v.R; ++i)
            if (v.n[i] == 1) dec_keys += (double)v.c[i] + 1 - (double)sc.pre_end[i] * B;
        const double sk_us = dec_keys * H_kv * 4.0 * d / kHbmBytesPerUs;
        if (ipr == kTcRows) {
            // Beside a decode pass that outlasts them twice over, 256-row items even
            // on a sparse grid: half the CTAs, each needing a whole SM, so split-K
            // keeps more SMs while the tiles run (c1_long: 0.481 -> 0.457 ms; c1, c3
            // unchanged within noise)
            double chain = 0;
            for (int i = 0; i < v.R; ++i)
                if (v.n[i] > 1)
                    chain = std::max(chain, (double)ceil_div((int64_t)v.c[i] + v.n[i], kTcKeys) * kTileUs);
            if (chain * 2 < sk_us) ipr = 2 * kTcRows;
        }
        // (never under a fixed split, o.split_tokens > 0: that mode promises a plan
        // independent of load and head count, so a KV-head slice is bit-identical, R17)
        if (o.split_prefill && o.split_tokens <= 0) {
            // pieces no longer than the longest of: the decode pass, the grid's
            // average load with every item whole, and 8 tiles
            double total_us = 0;
            for (int i = 0; i < v.R; ++i)
                if (v.n[i] > 1)
                    total_us += (double)H_kv * ceil_div((int64_t)v.n[i] * G, 2 * kTcRows) *
                                ceil_div((int64_t)v.c[i] + v.n[i], kTcKeys) * kTileUs;
            for (const Scratch::Node &nd : sc.nodes)
                if (nodes_tc) total_us += (double)H_kv * ceil_div((int64_t)nd.nm * G, 2 * kTcRows) *
                            ceil_div((int64_t)(nd.e - nd.a) * B, kTcKeys) * kTileUs;
            const double target_us = std::max({sk_us, total_us / o.num_sms, 8 * kTileUs});
            bool any = false;
            for (int i = 0; i < v.R; ++i)
                if (v.n[i] > 1) {
                    const double chain_us = (double)ceil_div((int64_t)v.c[i] + v.n[i], kTcKeys) * kTileUs;
                    // only a clear long pole pays for the partials and the merge
                    // (p1: a 78 us chain over a 70 us average -- cutting cost 25 us)
                    const int want = chain_us > 1.5 * target_us ? (int)std::ceil(chain_us / target_us - 1e-9) : 1;
                    sc.np[i] = std::max(1, std::min({want, kMaxCuts, 1 + v.c[i] / (2 * kTcKeys)}));
                    any |= sc.np[i] > 1;
                }
            if (any) ipr = 2 * kTcRows;
        }
    }
    // algorithmic unique KV tokens U: every shared block counted once
    {
        int64_t U = 0;
        for (int i = 0; i < v.R; ++i) U += (int64_t)v.c[i] + v.n[i] - (int64_t)v.s[i] * B;
        U += sc.n_shared * B;
        p->kv_bytes_unique = 4ll * d * H_kv * U;
    }
    int64_t kv_tok_read = 0;

    // ---- tcgen05 tiles: prefill chunks (n_i > 1), token-major stacking ----------
    if (tc_on) {
        for (int i = 0; i < v.R; ++i) {
            if (v.n[i] <= 1) continue;
            const int rows = v.n[i] * G;
            // key-range cuts of request i (sc.np[i] > 1): multiples of kTcKeys inside
            // its first c_i keys, spreading the ~ceil((c_i + n_i) / 128) tiles evenly
            int np = sc.np[i];
            int32_t cut[kMaxCuts + 1];
            if (np > 1) {
                const int64_t nt = ceil_div((int64_t)v.c[i] + v.n[i], kTcKeys), tc_full = v.c[i] / kTcKeys;
                np = std::min(np, kMaxCuts);
                int m = 0;
                cut[m++] = 0;
                for (int k = 1; k < np; ++k) {
                    const int64_t b = std::min<int64_t>((nt * k + np / 2) / np, tc_full) * kTcKeys;
                    if (b > cut[m - 1]) cut[m++] = (int32_t)b;
                }
                np = m;
            }
            if (np > 1) {
                for (int j = 0; j < v.n[i]; ++j) {
                    const int t = p->reqs[i].cu_q + j;
                    p->tok[t] = TokDev{(int32_t)p->n_slots, np, i, 0};
                    p->n_slots += (int64_t)np * G * H_kv;
                    p->comb.push_back(t);
                }
            }
            for (int g = 0; g < H_kv; ++g) {
                for (int r0 = 0; r0 < rows; r0 += ipr) {
                    const int nr = std::min(ipr, rows - r0);
                    const int j0 = r0 / G, j_last = (r0 + nr - 1) / G;
                    TcItem it{p->reqs[i].bt_off, g, 0, v.c[i] + j_last + 1, 0, p->reqs[i].cu_q + j0, nr, -1,
                              v.c[i] + j0, r0 - j0 * G, v.c[i]};
                    kv_tok_read += it.k1;
                    if (np == 1) {
                        p->tc.push_back(it);
                        continue;
                    }
                    for (int k = 0; k < np; ++k) {   // partial k of every row: keys [cut[k], cut[k+1] or k1)
                        TcItem pc = it;
                        pc.k0 = cut[k];
                        pc.k1 = k + 1 < np ? cut[k + 1] : it.k1;
                        pc.part = k;
                        p->tc.push_back(pc);
                    }
                }
            }
        }
    }
    // ---- split-K row chunks ----------------------------------------------------
    struct Chunk { int i, j0, nt, ks, ke; };
    std::vector<Chunk> ch_list;
    ch_list.reserve((size_t)v.R);
    const int tpi = std::max(1, kSkRows / G);
    int64_t total_keys = 0;
    for (int i = 0; i < v.R; ++i) {
        if (tc_on && v.n[i] > 1) continue;
        const int ks = sc.pre_end[i] * B;
        for (int j0 = 0; j0 < v.n[i]; j0 += tpi) {
            const int nt = std::min(tpi, v.n[i] - j0);
            Chunk ch{i, j0, nt, ks, v.c[i] + j0 + nt};
            total_keys += (int64_t)(ch.ke - ch.ks) * H_kv;
            ch_list.push_back(ch);
        }
    }
    // Persistent split-K grid (per KV head): CTA b runs items [sk_off[b], sk_off[b+1]).
    p->sk_off.assign(1, 0);
    auto add_tok_slots = [&](const Chunk &ch, int nparts) {
        if (nparts <= 1) return;
        for (int jj = 0; jj < ch.nt; ++jj) {
            const int t = p->reqs[ch.i].cu_q + ch.j0 + jj;
            p->tok[t] = TokDev{(int32_t)p->n_slots, nparts, ch.i, 0};
            p->n_slots += (int64_t)nparts * G * H_kv;
            p->comb.push_back(t);
        }
    };
    {
        int chunk_tok;
        if (o.split_tokens > 0) {
            chunk_tok = (o.split_tokens + B - 1) / B * B;
        } else {
            // ~one wave of split-K CTAs (3 resident per SM), LPT-ordered: fewer, longer
            // pieces than 4 waves' worth mean fewer partials to write and merge (c1
            // 0.451 -> 0.443 ms, its G = 8 shard 0.107 -> 0.099 ms; c2 / c3 within
            // 0.5 %); small batches keep the 256-key floor.  HG_SK_WAVES: A/B knob.
            static const double waves = getenv("HG_SK_WAVES") ? std::max(0.25, atof(getenv("HG_SK_WAVES"))) : 1.0;
            // split-K CTAs resident per SM (3 at the kernel's launch bounds); HG_SK_CTAS_PER_SM:
            // A/B knob for builds with a deeper ring (HG_SK_STAGES)
            static const int per_sm = getenv("HG_SK_CTAS_PER_SM") ? std::max(1, atoi(getenv("HG_SK_CTAS_PER_SM"))) : 3;
            const int64_t target = (int64_t)std::llround(o.num_sms * per_sm * waves);
            int64_t ct = (total_keys + target - 1) / std::max<int64_t>(target, 1);
            ct = std::max<int64_t>(ct, 256);
            chunk_tok = (int)((ct + B - 1) / B * B);
        }
        for (const Chunk &ch : ch_list) {
            const int pre = sc.npre[ch.i];
            const int pieces = std::max(1, ceil_div(ch.ke - ch.ks, chunk_tok));
            const int nparts = pre + pieces;
            add_tok_slots(ch, nparts);
            for (int k = 0; k < pieces; ++k) {
                const int k0 = ch.ks + k * chunk_tok;
                const int k1 = std::min(ch.ke, k0 + chunk_tok);
                // G_q > 16 (ch.nt == 1): the token's q heads in groups of 16 rows, each
                // item re-reading the same key range (adjacent in the LPT order: L2 hits)
                for (int h0 = 0; h0 < ch.nt * G; h0 += kSkRows)
                    p->sk.push_back(SkItem{ch.i, ch.j0, ch.nt, k0, k1, nparts > 1 ? pre + k : -1, h0,
                                           std::min(kSkRows, ch.nt * G - h0)});
                kv_tok_read += (int64_t)(k1 - k0) * H_kv * ((ch.nt * G + kSkRows - 1) / kSkRows);
            }
        }
    }
    // ---- prefix node tiles (partial `depth` of every member row): member-major stacking ----
    if (!sc.nodes.empty()) {
        int32_t off = 0;
        for (Scratch::Node &nd : sc.nodes) {
            nd.first = off;
            off += nd.nm;
            nd.nm = 0;
        }
        p->tc_tok.resize((size_t)off);
        for (int i = 0; i < v.R; ++i) {
            const int32_t *row = v.bt + (int64_t)i * v.W;
            for (int a = 0; a < sc.pre_end[i];) {
                Scratch::Node &nd = sc.nodes[sc.node[row[a]]];
                p->tc_tok[(size_t)nd.first + nd.nm++] = p->reqs[i].cu_q;
                a = nd.e;
            }
        }
        for (const Scratch::Node &nd : sc.nodes) {
            const int rows = nd.nm * G;
            if (!nodes_tc) {   // HBM route / route 3: 16-row split-K items over the node's keys (16 / G_q members each)
                const int mpi = kSkRows / G;
                for (int m0 = 0; m0 < nd.nm; m0 += mpi) {
                    const int nmm = std::min(mpi, nd.nm - m0);
                    p->sk.push_back(SkItem{nd.rep, nd.first + m0, nmm, nd.a * B, nd.e * B, nd.depth, 0, nmm * G, 1});
                    kv_tok_read += (int64_t)(nd.e - nd.a) * B * H_kv;
                    p->prefix_sk++;
                }
                continue;
            }
            for (int g = 0; g < H_kv; ++g) {
                for (int r0 = 0; r0 < rows; r0 += ipr) {
                    const int nr = std::min(ipr, rows - r0);
                    const int m0 = r0 / G;
                    TcItem it{p->reqs[nd.rep].bt_off, g, nd.a * B, nd.e * B, 1, nd.first + m0, nr, nd.depth, 0,
                              r0 - m0 * G, INT32_MAX};
                    kv_tok_read += (int64_t)(nd.e - nd.a) * B;
                    p->tc.push_back(it);
                    p->prefix_tiles++;
                }
            }
        }
    }
    p->kv_bytes_read = kv_tok_read * 4ll * d;
    // split-K: LPT order, one item per CTA (the hardware places them as SMs free up)
    lpt_sort(p->sk, p->sk_tmp);
    for (size_t k = 1; k <= p->sk.size(); ++k) p->sk_off.push_back((int32_t)k);
    // Persistent tcgen05 grid: one CTA per SM at most (each needs the SM's whole
    // shared memory); items beyond that are processed in LPT order by the same
    // CTAs without re-initialising the pipeline.  (Confining the tiles to a few
    // SMs beside the HBM-bound split-K kernel was measured slower: their K/V
    // loads queue behind split-K's HBM traffic.)
    p->tc_ctas = std::min((int)p->tc.size(), o.num_sms);
    stream_sort(p->tc, p->tc_tmp);
    assign_tc(p);

    // ---- workspace layout ----------------------------------------------------
    size_t off = 0;
    p->off_reqs = off;  off = align_up(off + sizeof(ReqDev) * p->reqs.size(), 16);
    p->off_bt = off;    off = align_up(off + sizeof(int32_t) * (size_t)p->n_bt, 16);
    p->off_sk = off;    off = align_up(off + sizeof(SkItem) * p->sk.size(), 16);
    p->off_tc = off;    off = align_up(off + sizeof(TcItem) * p->tc.size(), 16);
    p->off_rows = off;  off = align_up(off + sizeof(int32_t) * p->tc_tok.size(), 16);
    p->off_cbase = off; off = align_up(off + sizeof(TokDev) * p->tok.size(), 16);
    p->off_comb = off;  off = align_up(off + sizeof(int32_t) * p->comb.size(), 16);
    p->off_tcoff = off; off = align_up(off + sizeof(int32_t) * p->tc_off.size(), 16);
    p->off_skoff = off; off = align_up(off + sizeof(int32_t) * p->sk_off.size(), 16);
    // no tcgen05 item writes partials: split-K merges them itself (arrival counters,
    // zero in the uploaded image) and no combine kernel runs
    p->sk_merge = !p->comb.empty() && std::none_of(p->tc.begin(), p->tc.end(), [](const TcItem &it) { return it.part >= 0; });
    p->off_cnt = off;   off = align_up(off + (p->sk_merge ? sizeof(uint32_t) * (size_t)T * H_kv : 0), 16);
    p->off_exit = off;  off = align_up(off + 16, 16);   // split-K's entry / exit tickets (folded barriers)
    p->desc_bytes = off;   // the descriptor image lives in a library-owned device slot (api.cpp stage_desc)
    off = 0;               // the caller's workspace: partials and the rotated-Q copy only
    p->off_part_o = off;   off = align_up(off + sizeof(float) * (size_t)p->n_slots * d, 256);
    p->off_part_lse = off; off = align_up(off + sizeof(float) * (size_t)p->n_slots, 256);
    p->off_qrot = off;     off = align_up(off + (size_t)T * H_q * d * 2, 256);   // rotated Q (rope step)
    p->total_bytes = std::max<size_t>(off, 256);
    return HG_OK;
}

}  // namespace hg

// ---------------------------------------------------------------------------
// C ABI: pure host entry points
// ---------------------------------------------------------------------------
using namespace hg;

extern "C" const char *hg_last_error(void) { return g_err; }

extern "C" int32_t hg_get_num_blocks(int32_t tokens, int32_t block_size) {
    if (block_size < 1) return -1;
    if (tokens <= 0) return 0;
    return (int32_t)(((int64_t)tokens + block_size - 1) / block_size);
}
