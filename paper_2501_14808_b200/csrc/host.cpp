// host.cpp -- host-side steps of the hot path:
// error reporting, batch validation (§8(b) rules), prefix groups, and the
// per-call work plan consumed by the sm_100a kernels.
#include <algorithm>
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

// Stamp table reused across calls (per thread): detects duplicate ids in a row
// and ids shared outside the declared prefixes in one pass over the ids.
struct Stamp {
    std::vector<uint64_t> tag;  // epoch << 32 | row << 12 | col ... packed below
    uint32_t epoch = 0;
};
static thread_local Stamp g_stamp;

hg_status validate(const BatchView &v, int B, int num_blocks, int num_q_heads, int H_kv,
                   bool append) {
    if (num_q_heads >= 0) {
        if (H_kv <= 0 || num_q_heads <= 0 || num_q_heads % H_kv)
            return fail(HG_E_INVALID, "num_q_heads %d not a positive multiple of num_kv_heads %d",
                        num_q_heads, H_kv);
    }
    Stamp &st = g_stamp;
    if ((int)st.tag.size() < num_blocks) st.tag.assign((size_t)num_blocks, 0);
    if (++st.epoch == 0) {  // wrapped: clear
        std::fill(st.tag.begin(), st.tag.end(), 0);
        st.epoch = 1;
    }
    const uint64_t ep = (uint64_t)st.epoch << 40;
    int shared_write = -1;  // reported only if every INVALID rule passes
    for (int i = 0; i < v.R; ++i) {
        int64_t c = v.c[i], n = v.n[i], s = v.s[i];
        if (n < 1 || c < 0 || s < 0)
            return fail(HG_E_INVALID, "request %d: need n>=1, c>=0, s>=0 (c=%lld n=%lld s=%lld)", i,
                        (long long)c, (long long)n, (long long)s);
        int nb = ceil_div(c + n, B);
        if (nb > v.W) return fail(HG_E_INVALID, "request %d needs %d blocks > max_blocks_per_req %d", i, nb, v.W);
        if (s > nb) return fail(HG_E_INVALID, "request %d: shared blocks %lld > blocks %d", i, (long long)s, nb);
        if (append && c < s * B && shared_write < 0) shared_write = i;
        const int32_t *row = v.bt + (int64_t)i * v.W;
        for (int col = 0; col < nb; ++col) {
            int32_t b = row[col];
            if (b < 0 || b >= num_blocks)
                return fail(HG_E_INVALID, "request %d block %d: id %d outside [0, %d)", i, col, b, num_blocks);
            uint64_t t = st.tag[b];
            if ((t & ~((1ull << 40) - 1)) == ep) {
                int prow = (int)((t >> 16) & 0xFFFFFF), pcol = (int)(t & 0xFFFF);
                if (prow == i) return fail(HG_E_INVALID, "request %d lists block %d twice", i, b);
                if (col >= s || pcol >= v.s[prow])
                    return fail(HG_E_INVALID, "block %d used by requests %d and %d outside their shared prefixes",
                                b, prow, i);
            } else {
                st.tag[b] = ep | ((uint64_t)i << 16) | (uint64_t)col;
            }
        }
    }
    // equal first shared id => identical shared sequences
    for (int i = 0; i < v.R; ++i) {
        if (v.s[i] <= 0) continue;
        const int32_t *row = v.bt + (int64_t)i * v.W;
        uint64_t t = st.tag[row[0]];
        int prow = (int)((t >> 16) & 0xFFFFFF);
        if (prow == i) continue;  // i is the first user of this id
        const int32_t *prow_p = v.bt + (int64_t)prow * v.W;
        if (v.s[prow] != v.s[i] || memcmp(prow_p, row, sizeof(int32_t) * (size_t)v.s[i]) != 0 ||
            (t & 0xFFFF) != 0)
            return fail(HG_E_INVALID, "requests %d and %d share block %d but not an identical prefix", prow, i,
                        row[0]);
    }
    if (shared_write >= 0)
        return fail(HG_E_SHARED_WRITE, "request %d appends at position %d inside its shared prefix (%d blocks)",
                    shared_write, v.c[shared_write], v.s[shared_write]);
    return HG_OK;
}

void prefix_groups(const BatchView &v, std::vector<int32_t> *group) {
    // After validate(): the first user of a request's first shared id defines the group.
    group->assign((size_t)v.R, -1);
    std::vector<int32_t> first_of(v.R, -1);
    int ng = 0;
    Stamp &st = g_stamp;
    for (int i = 0; i < v.R; ++i) {
        if (v.s[i] <= 0) continue;
        int prow = (int)((st.tag[v.bt[(int64_t)i * v.W]] >> 16) & 0xFFFFFF);
        if (prow == i || (*group)[prow] < 0) {
            if ((*group)[prow] < 0) (*group)[prow] = ng++;
        }
        (*group)[i] = (*group)[prow];
    }
}

static size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

hg_status build_plan(const BatchView &v, int H_q, int H_kv, int d, const PlanOpts &o, Plan *p) {
    const int G = H_q / H_kv;
    const int B = kBlock;
    p->R = v.R;
    p->W = v.W;
    p->reqs.resize((size_t)v.R);
    p->sk.clear();
    p->tc.clear();
    p->tc_rows.clear();
    p->comb.clear();
    p->n_slots = 0;
    p->prefix_tiles = 0;
    int64_t T = 0, nbt = 0;
    for (int i = 0; i < v.R; ++i) {
        p->reqs[i] = ReqDev{v.c[i], v.n[i], (int32_t)T, (int32_t)nbt};
        T += v.n[i];
        nbt += ceil_div((int64_t)v.c[i] + v.n[i], B);
    }
    p->T = (int)T;
    p->bt_flat.resize((size_t)nbt);
    for (int i = 0; i < v.R; ++i) {
        int nb = ceil_div((int64_t)v.c[i] + v.n[i], B);
        memcpy(p->bt_flat.data() + p->reqs[i].bt_off, v.bt + (int64_t)i * v.W, sizeof(int32_t) * nb);
    }
    p->comb_base.assign((size_t)T * H_kv, -1);

    std::vector<int32_t> group;
    prefix_groups(v, &group);
    // prefix pass: groups with >= 2 decode members (a lone member gains nothing)
    const bool tc_ok = o.use_tc && tc_supported(d) && G <= kTcRows;
    std::vector<int32_t> gcount;
    for (int i = 0; i < v.R; ++i)
        if (group[i] >= 0 && v.n[i] == 1) {
            if ((int)gcount.size() <= group[i]) gcount.resize(group[i] + 1, 0);
            gcount[group[i]]++;
        }
    auto in_prefix_pass = [&](int i) {
        return o.prefix_pass && tc_ok && group[i] >= 0 && v.n[i] == 1 && gcount[group[i]] >= 2;
    };
    // algorithmic unique KV tokens U
    {
        int64_t U = 0;
        std::vector<char> seen(gcount.size() + 1, 0);
        std::vector<int32_t> gtok;
        for (int i = 0; i < v.R; ++i) {
            U += (int64_t)v.c[i] + v.n[i];
            if (group[i] >= 0) {
                if ((int)gtok.size() <= group[i]) gtok.resize(group[i] + 1, 0);
                if (seen.size() <= (size_t)group[i]) seen.resize(group[i] + 1, 0);
                if (seen[group[i]]) U -= (int64_t)v.s[i] * B;
                seen[group[i]] = 1;
            }
        }
        p->kv_bytes_unique = 4ll * d * H_kv * U;
    }
    int64_t kv_tok_read = 0;

    // ---- tcgen05 tiles: prefill chunks (n_i > 1) -------------------------------
    if (tc_ok) {
        for (int i = 0; i < v.R; ++i) {
            if (v.n[i] <= 1) continue;
            const int64_t rows = (int64_t)v.n[i] * G;
            for (int g = 0; g < H_kv; ++g) {
                for (int64_t r0 = 0; r0 < rows; r0 += kTcRows) {
                    int nr = (int)std::min<int64_t>(kTcRows, rows - r0);
                    int j_last = (int)((r0 + nr - 1) / G);
                    TcItem it{p->reqs[i].bt_off, g, 0, v.c[i] + j_last + 1, (int32_t)p->tc_rows.size(), nr, -1, 0};
                    for (int r = 0; r < nr; ++r) {
                        int j = (int)((r0 + r) / G), hl = (int)((r0 + r) % G);
                        p->tc_rows.push_back(TcRow{p->reqs[i].cu_q + j, g * G + hl, v.c[i] + j + 1, 0});
                    }
                    kv_tok_read += it.k1;
                    p->tc.push_back(it);
                }
            }
        }
    }
    // ---- split-K row chunks ----------------------------------------------------
    struct Chunk { int i, j0, nt, ks, ke; };
    std::vector<Chunk> chunks;
    const int tpi = std::max(1, kSkRows / G);
    int64_t total_keys = 0;
    for (int i = 0; i < v.R; ++i) {
        if (tc_ok && v.n[i] > 1) continue;
        int ks = in_prefix_pass(i) ? v.s[i] * B : 0;
        for (int j0 = 0; j0 < v.n[i]; j0 += tpi) {
            int nt = std::min(tpi, v.n[i] - j0);
            Chunk ch{i, j0, nt, ks, v.c[i] + j0 + nt};
            total_keys += (int64_t)(ch.ke - ch.ks) * H_kv;
            chunks.push_back(ch);
        }
    }
    int chunk_tok;
    if (o.split_tokens > 0) {
        chunk_tok = (o.split_tokens + B - 1) / B * B;
    } else {
        const int64_t target = (int64_t)o.num_sms * 3 * 4;
        int64_t ct = (total_keys + target - 1) / std::max<int64_t>(target, 1);
        ct = std::max<int64_t>(ct, 256);
        chunk_tok = (int)((ct + B - 1) / B * B);
    }
    // prefix group tiles (part 0 of every member row)
    std::vector<std::vector<int>> members(gcount.size());
    for (int i = 0; i < v.R; ++i)
        if (in_prefix_pass(i)) members[group[i]].push_back(i);
    for (int i = 0; i < v.R; ++i) (void)i;
    // partial slots for split-K rows
    for (const Chunk &ch : chunks) {
        const int pre = in_prefix_pass(ch.i) ? 1 : 0;
        const int pieces = std::max(1, ceil_div(ch.ke - ch.ks, chunk_tok));
        const int nparts = pre + pieces;
        std::vector<int32_t> bases(ch.nt, -1);
        for (int g = 0; g < H_kv; ++g) {
            if (nparts > 1) {
                for (int jj = 0; jj < ch.nt; ++jj) {
                    int t = p->reqs[ch.i].cu_q + ch.j0 + jj;
                    int32_t base = (int32_t)p->n_slots;
                    p->n_slots += (int64_t)nparts * G;
                    p->comb_base[(size_t)t * H_kv + g] = base;
                    p->comb.push_back(CombItem{t, g, base, nparts});
                }
            }
            for (int k = 0; k < pieces; ++k) {
                int k0 = ch.ks + k * chunk_tok;
                int k1 = std::min(ch.ke, k0 + chunk_tok);
                p->sk.push_back(SkItem{ch.i, g, ch.j0, ch.nt, k0, k1, nparts > 1 ? pre + k : -1, 0});
                kv_tok_read += (k1 - k0);
            }
        }
    }
    for (size_t gi = 0; gi < members.size(); ++gi) {
        const auto &mem = members[gi];
        if (mem.empty()) continue;
        const int P = v.s[mem[0]] * B;
        const int64_t rows = (int64_t)mem.size() * G;
        for (int g = 0; g < H_kv; ++g) {
            for (int64_t r0 = 0; r0 < rows; r0 += kTcRows) {
                int nr = (int)std::min<int64_t>(kTcRows, rows - r0);
                TcItem it{p->reqs[mem[0]].bt_off, g, 0, P, (int32_t)p->tc_rows.size(), nr, 0, 0};
                for (int r = 0; r < nr; ++r) {
                    int m = (int)((r0 + r) / G), hl = (int)((r0 + r) % G);
                    p->tc_rows.push_back(TcRow{p->reqs[mem[m]].cu_q, g * G + hl, P, 0});
                }
                kv_tok_read += P;
                p->tc.push_back(it);
                p->prefix_tiles++;
            }
        }
    }
    p->kv_bytes_read = kv_tok_read * 4ll * d;
    // LPT order: longest key ranges first
    std::stable_sort(p->sk.begin(), p->sk.end(),
                     [](const SkItem &a, const SkItem &b) { return (a.k1 - a.k0) > (b.k1 - b.k0); });
    std::stable_sort(p->tc.begin(), p->tc.end(),
                     [](const TcItem &a, const TcItem &b) { return (a.k1 - a.k0) > (b.k1 - b.k0); });

    // ---- workspace layout ----------------------------------------------------
    size_t off = 0;
    p->off_reqs = off;  off = align_up(off + sizeof(ReqDev) * p->reqs.size(), 16);
    p->off_bt = off;    off = align_up(off + sizeof(int32_t) * p->bt_flat.size(), 16);
    p->off_sk = off;    off = align_up(off + sizeof(SkItem) * p->sk.size(), 16);
    p->off_tc = off;    off = align_up(off + sizeof(TcItem) * p->tc.size(), 16);
    p->off_rows = off;  off = align_up(off + sizeof(TcRow) * p->tc_rows.size(), 16);
    p->off_cbase = off; off = align_up(off + sizeof(int32_t) * p->comb_base.size(), 16);
    p->off_comb = off;  off = align_up(off + sizeof(CombItem) * p->comb.size(), 16);
    p->desc_bytes = off;
    off = align_up(off, 256);
    p->off_part_o = off;   off = align_up(off + sizeof(float) * (size_t)p->n_slots * d, 256);
    p->off_part_lse = off; off = align_up(off + sizeof(float) * (size_t)p->n_slots, 256);
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
