// psm.cpp -- Prefix Sharing Maximization (HyGen §4.3; Alg. 3,
// P:534-583): offline requests live in a prefix tree T_p
// over their prompt tokens; the offline phase admits them in the tree's DFS
// order, so requests that share a prefix land in the same batch and their
// prefix KV can be shared (the prefix-group pass of hg_hybrid_attention).
//
// DFS order: at a node, the requests whose prompt ends there (insertion order),
// then the children in order of first insertion.  The DFS list is rebuilt
// lazily after inserts; removal is O(1) (marks + counts), matching the paper's
// "pre-processed list ... synced up with the prefix tree".
#include <algorithm>
#include <unordered_map>
#include <vector>

#include "hg_internal.h"

using namespace hg;

struct hg_psm {
    struct Node {
        std::vector<std::pair<int32_t, int32_t>> kids;  // (token, node) in first-insertion order
        std::unordered_map<int32_t, int32_t> index;     // token -> node
        std::vector<int32_t> reqs;                       // requests ending here
        int32_t depth = 0;
    };
    std::vector<Node> nodes{1};
    std::unordered_map<int32_t, int32_t> where;          // request -> node
    std::unordered_map<int32_t, char> alive;
    std::vector<int32_t> order, order_depth;              // DFS list (request, depth of its node)
    std::vector<int32_t> lcp;                            // LCP with the DFS predecessor
    bool dirty = false;
    int32_t live = 0;

    void rebuild() {
        order.clear();
        lcp.clear();
        // iterative preorder; track, for every emitted request, the depth of the
        // deepest common ancestor with the previously emitted request
        struct Frame { int32_t node, next_kid; };
        std::vector<Frame> st{{0, 0}};
        int32_t min_depth_since = 0;  // shallowest node on the path walked since the last emitted request
        bool first = true;
        std::vector<char> seen_node(nodes.size(), 0);
        while (!st.empty()) {
            Frame &f = st.back();
            Node &n = nodes[f.node];
            if (!seen_node[f.node]) {
                seen_node[f.node] = 1;
                for (int32_t r : n.reqs) {
                    if (!alive.count(r)) continue;
                    order.push_back(r);
                    lcp.push_back(first ? 0 : min_depth_since);
                    first = false;
                    min_depth_since = n.depth;
                }
            }
            if (f.next_kid < (int32_t)n.kids.size()) {
                const int32_t child = n.kids[f.next_kid++].second;
                st.push_back({child, 0});
            } else {
                st.pop_back();
                if (!st.empty()) min_depth_since = std::min(min_depth_since, nodes[st.back().node].depth);
            }
        }
        dirty = false;
    }
};

extern "C" hg_status hg_psm_create(hg_psm **out) {
    if (!out) return fail(HG_E_INVALID, "NULL argument");
    *out = new hg_psm();
    return HG_OK;
}

extern "C" hg_status hg_psm_destroy(hg_psm *p) {
    delete p;
    return HG_OK;
}

extern "C" hg_status hg_psm_insert(hg_psm *p, int32_t rid, const int32_t *tokens, int32_t n) {
    if (!p || n < 0 || (n > 0 && !tokens)) return fail(HG_E_INVALID, "bad arguments");
    if (p->where.count(rid)) return fail(HG_E_INVALID, "request %d already in the prefix tree", rid);
    int32_t cur = 0;
    for (int32_t k = 0; k < n; ++k) {
        auto it = p->nodes[cur].index.find(tokens[k]);
        if (it == p->nodes[cur].index.end()) {
            const int32_t nn = (int32_t)p->nodes.size();
            p->nodes.emplace_back();
            p->nodes[nn].depth = p->nodes[cur].depth + 1;
            p->nodes[cur].index.emplace(tokens[k], nn);
            p->nodes[cur].kids.push_back({tokens[k], nn});
            cur = nn;
        } else {
            cur = it->second;
        }
    }
    p->nodes[cur].reqs.push_back(rid);
    p->where[rid] = cur;
    p->alive[rid] = 1;
    p->live++;
    p->dirty = true;
    return HG_OK;
}

extern "C" hg_status hg_psm_remove(hg_psm *p, int32_t rid) {
    if (!p) return fail(HG_E_INVALID, "NULL argument");
    auto it = p->alive.find(rid);
    if (it == p->alive.end()) return fail(HG_E_INVALID, "request %d not in the prefix tree", rid);
    p->alive.erase(it);
    auto &v = p->nodes[p->where[rid]].reqs;
    v.erase(std::find(v.begin(), v.end(), rid));
    p->where.erase(rid);
    p->live--;
    p->dirty = true;
    return HG_OK;
}

extern "C" int32_t hg_psm_size(const hg_psm *p) { return p ? p->live : 0; }

extern "C" hg_status hg_psm_dfs_order(hg_psm *p, int32_t *ids, int32_t *lcp, int32_t max, int32_t *n_out) {
    if (!p || !n_out || max < 0 || (max > 0 && !ids)) return fail(HG_E_INVALID, "bad arguments");
    if (p->dirty) p->rebuild();
    const int32_t n = std::min<int32_t>(max, (int32_t)p->order.size());
    for (int32_t k = 0; k < n; ++k) {
        ids[k] = p->order[k];
        if (lcp) lcp[k] = p->lcp[k];
    }
    *n_out = n;
    return HG_OK;
}
