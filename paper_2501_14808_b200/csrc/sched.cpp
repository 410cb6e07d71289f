// sched.cpp -- SLO_AWARE_SCHEDULE of HyGen Alg. 1 over the
// fitted batch-latency predictor: the batch composer that
// drives hg_hybrid_attention each iteration.
//
// Readings (R19-R21):
//  * t_req of a request is its marginal batch-latency increase
//    predict(B + r) - predict(B) under the linear model, clamped at 0; the
//    intercept w[0] is charged once, before the first request (t <- t - w0).
//  * get_max_tokens(t, c, m, r) = largest l <= min(c, prompt_left(r), m*B) whose
//    marginal fits t (exact: binary search when the model is monotone in l,
//    i.e. the S_p, S_p^2 and P2 weights are >= 0; a downward scan otherwise).
//  * PERFORM_PREEMPTION is not modelled (preemption is out of scope): a prefill
//    that does not fit ends the pass in both phases (Alg. 1's `break`).
//  * Online decodes are admitted unconditionally and still decrement t.
#include <algorithm>
#include <cmath>
#include <vector>

#include "hg_internal.h"

using namespace hg;

namespace {
struct Acc {   // batch features under construction, in the hg_features order
    double f[8] = {0, 0, 0, 0, 0, 0, 0, 0};
};
double lin(const hg_predictor &m, const double *f) {
    double a = 0;
    for (int k = 0; k < 8; ++k) a += m.w[1 + k] * f[k];
    return a;
}
// features after adding one decode row of context c (shared prefix s_tok counted once per group)
void add_decode(const Acc &a, int c, int s_tok_dup, double *out) {
    for (int k = 0; k < 8; ++k) out[k] = a.f[k];
    out[1] += 1;                                   // S_d
    out[3] = out[1] * out[1];                      // S_d^2
    out[5] += 1;                                   // N_d
    out[7] += (double)(c + 1) - s_tok_dup;         // D_ctx (unique KV tokens)
}
void add_prefill(const Acc &a, int c, int l, double *out) {
    for (int k = 0; k < 8; ++k) out[k] = a.f[k];
    out[0] += l;                                   // S_p
    out[2] = out[0] * out[0];                      // S_p^2
    out[4] += 1;                                   // N_p
    out[6] += (double)l * ((double)c + (double)(l + 1) / 2.0);  // P2
}
// The batch under construction across the calls of one iteration (Alg. 2 runs
// the online then the offline phase on ONE batch): its features,
// whether the intercept was charged, and the groups that already have a decode
// row.  Loaded from / stored to the caller's hg_sched_state (NULL: a fresh
// batch, intercept charged in this call).
struct Batch {
    Acc acc;
    std::vector<int32_t> groups_in;
    hg_sched_state *st = nullptr;
    hg_status load(hg_sched_state *s, const hg_predictor &M, double *t) {
        st = s;
        if (s) {
            if (s->n_groups < 0 || s->n_groups > HG_SCHED_MAX_GROUPS) return fail(HG_E_INVALID, "state.n_groups");
            for (int k = 0; k < 8; ++k) acc.f[k] = s->features[k];
            groups_in.assign(s->groups, s->groups + s->n_groups);
            if (s->intercept_charged) return HG_OK;
        }
        *t -= M.w[0];   // the batch's fixed cost (intercept) is charged once per batch
        return HG_OK;
    }
    hg_status store() {
        if (!st) return HG_OK;
        if (groups_in.size() > (size_t)HG_SCHED_MAX_GROUPS)
            return fail(HG_E_UNSUPPORTED, "more than %d shared-prefix groups in one batch", HG_SCHED_MAX_GROUPS);
        for (int k = 0; k < 8; ++k) st->features[k] = acc.f[k];
        st->intercept_charged = 1;
        st->n_groups = (int32_t)groups_in.size();
        std::copy(groups_in.begin(), groups_in.end(), st->groups);
        return HG_OK;
    }
    bool has_group(int32_t g) const { return std::find(groups_in.begin(), groups_in.end(), g) != groups_in.end(); }
};
}  // namespace

extern "C" hg_status hg_slo_aware_schedule(const hg_predictor *model, int32_t block_size, const hg_sched_req *running,
                                           int32_t n_running, const hg_sched_req *queue, int32_t n_queue,
                                           double t_budget, int32_t chunk_budget, int32_t memory_blocks,
                                           int32_t phase_online, hg_sched_state *state, hg_sched_entry *out,
                                           int32_t *n_out, double *t_left, int32_t *c_left, int32_t *m_left) {
    if (!model || block_size < 1 || n_running < 0 || n_queue < 0 || (n_running && !running) || (n_queue && !queue) ||
        !out || !n_out || chunk_budget < 0 || memory_blocks < 0)
        return fail(HG_E_INVALID, "bad arguments");
    const hg_predictor &M = *model;
    double t = t_budget;
    Batch bat;
    hg_status st = bat.load(state, M, &t);
    if (st) return st;
    int64_t c = chunk_budget, m = memory_blocks;
    int nb = 0;
    Acc &acc = bat.acc;
    std::vector<int32_t> &groups_in = bat.groups_in;   // shared-prefix groups that already have a decode row in B
    double f[8];
    auto marginal = [&](const double *fn) { return std::max(0.0, lin(M, fn) - lin(M, acc.f)); };
    // ---- decodes of the running requests (Alg. 1 lines 6-13) ----
    for (int i = 0; i < n_running; ++i) {
        const hg_sched_req &r = running[i];
        if (r.prompt_left > 0) continue;
        const int dup = r.group >= 0 && r.shared_prefix_tokens > 0 && bat.has_group(r.group) ? r.shared_prefix_tokens : 0;
        add_decode(acc, r.cached, dup, f);
        const double t_req = marginal(f);
        if (t_req <= t || phase_online) {
            t -= t_req;
            for (int k = 0; k < 8; ++k) acc.f[k] = f[k];
            if (r.group >= 0 && r.shared_prefix_tokens > 0 && !dup) groups_in.push_back(r.group);
            out[nb++] = hg_sched_entry{i, 0, t_req};
        }
    }
    // ---- prefilling requests, then the queue (lines 14-33) ----
    const bool monotone = M.w[1 + 0] >= 0 && M.w[1 + 2] >= 0 && M.w[1 + 6] >= 0;
    const int n_all = n_running + n_queue;
    for (int k = 0; k < n_all; ++k) {
        const hg_sched_req &r = k < n_running ? running[k] : queue[k - n_running];
        if (k < n_running && r.prompt_left <= 0) continue;   // decodes were handled above
        if (r.prompt_left <= 0) continue;                    // a queued request with nothing to prefill
        // get_max_tokens(t, c, m, r)
        const int64_t hi = std::min<int64_t>(std::min<int64_t>(c, r.prompt_left), m * (int64_t)block_size);
        auto fits = [&](int64_t l, double *t_req) {
            add_prefill(acc, r.cached, (int)l, f);
            *t_req = marginal(f);
            return *t_req <= t;
        };
        int64_t l = 0;
        double t_req = 0;
        if (hi > 0) {
            double tr;
            if (fits(hi, &tr)) {
                l = hi;
                t_req = tr;
            } else if (monotone) {
                int64_t lo = 0, up = hi;   // fits(lo) (or lo == 0), !fits(up)
                while (up - lo > 1) {
                    const int64_t mid = (lo + up) / 2;
                    if (fits(mid, &tr)) lo = mid; else up = mid;
                }
                l = lo;
                if (l > 0) fits(l, &t_req);
            } else {
                for (int64_t cand = hi - 1; cand >= 1; --cand)
                    if (fits(cand, &tr)) { l = cand; t_req = tr; break; }
            }
        }
        if (l > 0) {
            add_prefill(acc, r.cached, (int)l, f);
            for (int q = 0; q < 8; ++q) acc.f[q] = f[q];
            t -= t_req;
            c -= l;
            m -= hg_get_num_blocks((int32_t)l, block_size);   // GET_NUM_BLOCKS(l)
            out[nb++] = hg_sched_entry{k, (int32_t)l, t_req};
        } else {
            break;   // (online: PERFORM_PREEMPTION + retry is out of scope, reading R21)
        }
    }
    st = bat.store();
    if (st) return st;
    *n_out = nb;
    if (t_left) *t_left = t;
    if (c_left) *c_left = (int32_t)c;
    if (m_left) *m_left = (int32_t)m;
    return HG_OK;
}

// ---------------------------------------------------------------------------
// Alg. 3 PREFIX_SHARING_OFFLINE_SCHEDULE: running offline requests
// in their order (decode: stop at the first that does not fit -- reading R16
// of the inverted `IF t > t_req THEN break`; prefill: largest fitting chunk or
// stop), then new requests in the prefix tree's DFS order (T_p.get_next_request),
// each removed from the tree once scheduled.
// ---------------------------------------------------------------------------
extern "C" hg_status hg_psm_offline_schedule(const hg_predictor *model, int32_t block_size, hg_psm *psm,
                                             const hg_sched_req *running, int32_t n_running,
                                             const hg_sched_req *by_id, int32_t n_ids, double t_budget,
                                             int32_t chunk_budget, int32_t memory_blocks, hg_sched_state *state,
                                             hg_sched_entry *out, int32_t *n_out, double *t_left, int32_t *c_left,
                                             int32_t *m_left) {
    if (!model || !psm || block_size < 1 || n_running < 0 || (n_running && !running) || n_ids < 0 ||
        (n_ids && !by_id) || !out || !n_out || chunk_budget < 0 || memory_blocks < 0)
        return fail(HG_E_INVALID, "bad arguments");
    const hg_predictor &M = *model;
    double t = t_budget;
    Batch bat;
    hg_status st = bat.load(state, M, &t);
    if (st) return st;
    int64_t c = chunk_budget, m = memory_blocks;
    int nb = 0;
    Acc &acc = bat.acc;
    std::vector<int32_t> &groups_in = bat.groups_in;
    double f[8];
    auto marginal = [&](const double *fn) { return std::max(0.0, lin(M, fn) - lin(M, acc.f)); };
    const bool monotone = M.w[1 + 0] >= 0 && M.w[1 + 2] >= 0 && M.w[1 + 6] >= 0;
    auto max_prefill = [&](const hg_sched_req &r, double *t_req) -> int64_t {
        const int64_t hi = std::min<int64_t>(std::min<int64_t>(c, r.prompt_left), m * (int64_t)block_size);
        double tr;
        auto fits = [&](int64_t l) {
            add_prefill(acc, r.cached, (int)l, f);
            tr = marginal(f);
            return tr <= t;
        };
        if (hi <= 0) return 0;
        if (fits(hi)) { *t_req = tr; return hi; }
        int64_t l = 0;
        if (monotone) {
            int64_t lo = 0, up = hi;
            while (up - lo > 1) {
                const int64_t mid = (lo + up) / 2;
                if (fits(mid)) lo = mid; else up = mid;
            }
            l = lo;
        } else {
            for (int64_t cand = hi - 1; cand >= 1; --cand)
                if (fits(cand)) { l = cand; break; }
        }
        if (l > 0) { fits(l); *t_req = tr; }
        return l;
    };
    auto take_prefill = [&](const hg_sched_req &r, int64_t l, double t_req, int32_t index) {
        add_prefill(acc, r.cached, (int)l, f);
        for (int q = 0; q < 8; ++q) acc.f[q] = f[q];
        t -= t_req;
        c -= l;
        m -= hg_get_num_blocks((int32_t)l, block_size);
        out[nb++] = hg_sched_entry{index, (int32_t)l, t_req};
    };
    bool stopped = false;
    for (int i = 0; i < n_running && !stopped; ++i) {
        const hg_sched_req &r = running[i];
        if (r.prompt_left <= 0) {
            const int dup =
                r.group >= 0 && r.shared_prefix_tokens > 0 && bat.has_group(r.group) ? r.shared_prefix_tokens : 0;
            add_decode(acc, r.cached, dup, f);
            const double t_req = marginal(f);
            if (t < t_req) { stopped = true; break; }
            t -= t_req;
            for (int q = 0; q < 8; ++q) acc.f[q] = f[q];
            if (r.group >= 0 && r.shared_prefix_tokens > 0 && !dup) groups_in.push_back(r.group);
            out[nb++] = hg_sched_entry{i, 0, t_req};
        } else {
            double t_req = 0;
            const int64_t l = max_prefill(r, &t_req);
            if (l > 0) take_prefill(r, l, t_req, i);
            else stopped = true;
        }
    }
    while (!stopped && hg_psm_size(psm) > 0) {
        int32_t rid, n1 = 0;
        hg_status s = hg_psm_dfs_order(psm, &rid, nullptr, 1, &n1);
        if (s) return s;
        if (n1 == 0) break;
        if (rid < 0 || rid >= n_ids) return fail(HG_E_INVALID, "prefix-tree request %d has no entry in by_id", rid);
        const hg_sched_req &r = by_id[rid];
        double t_req = 0;
        const int64_t l = max_prefill(r, &t_req);
        if (l <= 0) break;
        take_prefill(r, l, t_req, n_running + rid);
        hg_psm_remove(psm, rid);
    }
    st = bat.store();
    if (st) return st;
    *n_out = nb;
    if (t_left) *t_left = t;
    if (c_left) *c_left = (int32_t)c;
    if (m_left) *m_left = (int32_t)m;
    return HG_OK;
}
